"""bench.py's JSON-line contract and measurement helpers, on CPU: the
compact line keeps every key the driver reads; the tensor roofline takes
the burst peak for sub-2 s regions and the sustained one beyond; a hybrid
GEMM's companion kernel on another stream folds into the launch it
overlaps; skipped optional launches are not counted."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def _out():
    roof = bench.gemm_roofline(
        [{"desc": "gemm tcgen05 bf16 %z1 M=65536", "ms": 1.6, "excl_ms": 1.6, "flops": 2.2e12, "bytes": 0,
          "timing": "cupti"},
         {"desc": "finalize %d15", "ms": 0.01, "excl_ms": 0.01, "flops": 0.0, "bytes": 0, "timing": "cupti"}],
        {"bf16_tflops": 1637.4, "bf16_tflops_sustained": 1362.7, "source": "MEASURED_PEAKS.json"}, 0.2)
    roof["traffic"] = 1.7e9
    return {"metric": bench.METRIC, "value": 6.6e6, "unit": "samples/s", "n_gpus": 1, "steps": 20, "warmup": 5,
            "ms_per_step": 9.9, "step_ms": {"p10": 9.0, "median": 10.1, "p90": 10.3}, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "c4_mlp", "global_batch": 65536, "per_rank_batch": 65536, "parallelism": "dp1",
                       "l2": "inputs larger than L2", "extra": "dropped"},
            "step_tflops": 1300.0, "gpu_launches": 300,
            "clocks": {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"]},
            "roofline": roof,
            "e2e": {"value": 6.0e6, "unit": "samples/s", "ms_per_step": 10.8, "h2d_bytes_per_step": 602406912,
                    "d2h_bytes_per_step": 4, "api": "dropped"},
            "cpu_baseline": {"value": 1000.0, "unit": "samples/s", "cores": 16, "kind": "oracle",
                             "sample": "128 rows"}}


def test_compact_line_keeps_the_contract_keys():
    line = bench.compact_line(_out())
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks", "roofline", "e2e", "cpu_baseline"):
        assert k in line, k
    assert line["config"]["workload"] == "c4_mlp" and "extra" not in line["config"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in line["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in line["e2e"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in line["cpu_baseline"], k
    assert set(line["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_roofline_peak_choice():
    kb = [{"desc": "gemm tcgen05 bf16 %z1", "ms": 1.0, "excl_ms": 1.0, "flops": 1.5e12, "bytes": 0, "timing": "cupti"}]
    pk = {"bf16_tflops": 1637.4, "bf16_tflops_sustained": 1362.7, "source": "x"}
    short = bench.gemm_roofline(kb, pk, 0.5)
    long_ = bench.gemm_roofline(kb, pk, 5.0)
    assert short["peak"] == 1637.4 and short["peak_kind"].startswith("burst")
    assert long_["peak"] == 1362.7 and long_["peak_kind"].startswith("sustained")
    assert abs(short["achieved"] - 1500.0) < 1e-6 and abs(short["frac"] - 1500.0 / 1637.4) < 1e-4


def test_hybrid_companion_kernels_fold_and_skipped_launches_do_not_count():
    R = bench._Rec
    ks = [R("gemm_tc_kernel A", 0, 100, 7), R("ew_kernel", 110, 5, 7), R("gemm_tc_kernel B", 5, 120, 9),
          R("gemm_tc_kernel C", 200, 50, 7)]
    m = bench._merge_hybrid(ks)
    assert [k.name for k in m] == ["gemm_tc_kernel A", "ew_kernel", "gemm_tc_kernel C"]
    assert m[0].start == 0 and m[0].dur == 125 and m[0].parts == 2 and m[2].parts == 1
    kb = [{"kernel": "gemm", "kernels": 2}, {"kernel": "(not launched)"}, {"kernel": "ew"}]
    assert bench.launched(kb) == 3
