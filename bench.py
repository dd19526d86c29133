#!/usr/bin/env python
"""Benchmark of the DLVM hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c3|c1|c2|c5]
    python bench.py --impl reference ...   # the CPU float64 oracle as the reference arm

Default workload (N GPUs, one process per GPU under torchrun): BASELINE.json
config 4 -- the c3 MLP 4096->4096->4096->1000 (ReLU, MSE) at global batch
65536, rows split over ranks, one fwd+adjoint step = dlvm_grad_run (forward
recomputed inside the generated gradient function) + the bucketed NCCL
gradient all-reduce.  Metric: global samples/s (strong scaling: fixed global
batch).  Rank 0 also measures config 2 (the fused element-wise chain on 2^28
fp32 elements) as `fused_elementwise` (HBM GB/s) when N == 1.

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
synchronize, CUDA events on the launching stream, max over ranks.  Inputs
are larger than L2 (x alone is 512 MiB per rank at N=1).  Per-kernel times
come from CUPTI kernel activity records in a separate short pass after the
timed region (PDL overlap intact); `roofline` reports the dominant kernel
(the longest GEMM) against the measured bf16 peak -- burst for timed regions
under 2 s, sustained beyond -- and the GEMM class from exclusive times.
`--gpus N` outside torchrun re-runs the command as N ranks under
torch.distributed.run.  Per-kernel lists go to a detail file (`--detail`).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MLP fwd+adjoint samples/s at 1/2/4/8 B200; fused-elementwise HBM GB/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None
        self.window = None  # (t0, t1) wall-clock seconds of the timed region

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(1.0)  # nvidia-smi start-up, so samples cover the timed region
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        """Median SM clock and active throttle reasons of the samples taken
        inside the timed window (all samples if the window caught none)."""
        import datetime
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def ts(r):
            try:
                return datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                return None

        inside = rows
        if self.window:
            t0, t1 = self.window
            w = [r for r in rows if ts(r) is not None and t0 - 0.06 <= ts(r) <= t1 + 0.06]
            if w:
                inside = w
        num = lambda x: x.replace(".", "", 1).isdigit()
        sm = [float(r[1]) for r in inside if num(r[1])]
        mx = [float(r[2]) for r in inside if num(r[2])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in inside for n, v in zip(names, r[5:9]) if v.lower().startswith("active")})
        pw = [float(r[3]) for r in inside if num(r[3])]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "samples_total": len(rows),
                "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------- workloads
def to_dev(x, dev, bf16=False):
    import torch
    t = torch.from_numpy(x).to(dev, non_blocking=False)
    return t.to(torch.bfloat16) if bf16 else t


def mlp_setup(w, dev, rank):
    """Inputs of the MLP gradient on this rank: x and W as bf16 (the bf16 dot
    policy rounds them anyway), one-hot t as bool bytes (0/1 values, exact),
    the rest f32 (dlvm.h storage rule).  Returns (handle, dev inputs, seed,
    host inputs, n_grads)."""
    import numpy as np
    import torch
    import paper_1711_03016_b200 as P
    f = P.Function(w.text, w.fn, w.grad, dot_precision=w.dot_precision)
    host = w.inputs(row_offset=rank * w.batch)
    dev_in = []
    for a, x in zip(w.args, host):
        # bf16 storage (dlvm.h): the dot operands the bf16 policy rounds anyway;
        # one-hot targets as bool bytes (exact) -- a quarter of their f32 upload in e2e
        bf = w.dot_precision == "bf16" and (a.name == "x" or a.name.startswith("w"))
        if a.dist[0] == "onehot":
            dev_in.append(torch.from_numpy(x != 0).to(dev))
        else:
            dev_in.append(to_dev(x, dev, bf))
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    return f, dev_in, seed, host, 2 * len(w.layers)


def time_steps(step, K, dev, world, group=None, stats=None):
    """K steps bracketed by barrier + synchronize; device time by CUDA events
    on the current stream; max over ranks.  Returns ms per step.  An event
    after every step (a marker: it does not synchronise) gives this rank's
    per-step times; with `stats` (a dict) their p10 / median / p90 go there
    (SURVEY 8(d) protocol)."""
    import torch
    import torch.distributed as dist
    st = torch.cuda.current_stream(dev)
    if world > 1:
        dist.barrier(group=group)
    torch.cuda.synchronize(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    ev[0].record(st)
    for k in range(K):
        step()
        ev[k + 1].record(st)
    torch.cuda.synchronize(dev)
    ms = ev[0].elapsed_time(ev[K]) / K
    if stats is not None and K > 0:
        per = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(K))
        q = lambda f: per[min(K - 1, int(round(f * (K - 1))))]
        stats.update({"p10": round(q(0.1), 4), "median": round(q(0.5), 4), "p90": round(q(0.9), 4)})
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        dist.barrier(group=group)
        ms = float(t.item())
    return ms


class _Rec:
    """One kernel activity record (name, start ns, duration ns, stream)."""

    def __init__(self, name, start, dur, stream):
        self.name, self.start, self.dur, self.stream = name, start, dur, stream
        self.parts = 1  # kernels folded into this record (a hybrid GEMM: 2)


def _merge_hybrid(ks):
    """A hybrid GEMM launch is two kernels: multicast clusters on the
    caller's stream and CTA pairs on an auxiliary stream (gemm_tc.cuh
    launch_hybrid).  Each GEMM kernel off the main stream (the stream most
    kernels ran on) is folded into the main-stream GEMM kernel it overlaps,
    which then spans both; the result is sorted by start time."""
    if not ks:
        return ks
    streams = [k.stream for k in ks]
    main = max(set(streams), key=streams.count)
    mains = sorted([k for k in ks if k.stream == main], key=lambda k: k.start)
    for c in (k for k in ks if k.stream != main):
        best, ov = None, 0
        for m in mains:
            o = min(m.start + m.dur, c.start + c.dur) - max(m.start, c.start)
            if "gemm_tc" in m.name and o > ov:
                best, ov = m, o
        if best is None:
            mains.append(c)  # not a companion: keep it as a launch of its own
            continue
        end = max(best.start + best.dur, c.start + c.dur)
        best.start = min(best.start, c.start)
        best.dur = end - best.start
        best.parts += c.parts
    return sorted(mains, key=lambda k: k.start)


def kernel_breakdown(f, which, step, K, dev):
    """Per-launch device times of K steps from CUPTI kernel activity records
    (torch.profiler / kineto), which -- unlike CUDA events recorded between
    launches -- leave programmatic dependent launch (PDL) overlap intact.
    For launch i: `ms` = mean CUPTI duration (start to end of the kernel,
    including any PDL wait at its griddepcontrol.wait) and `excl_ms` = the
    part of the step timeline it alone accounts for (end minus the later of
    its start and every earlier kernel's end), so the exclusive times of a
    step add up to its busy time.  Falls back to inter-launch events (marked
    `timing: events`) if the activity records do not match the plan."""
    import torch
    n = f.num_launches(which)
    out = None
    try:
        from torch.autograd import DeviceType
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize(dev)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(K + 1):  # the first step primes the tracer (its first kernel can be missed)
                step()
            torch.cuda.synchronize(dev)
        ks = [_Rec(e.name(), e.start_ns(), e.duration_ns(), e.device_resource_id())
              for e in prof.profiler.kineto_results.events()
              if e.device_type() == DeviceType.CUDA and any(k in e.name() for k in OWN_KERNELS)]
        ks = _merge_hybrid(ks)
        # match the plan's launches to the recorded kernels by kind, walking
        # back from the last step (a kernel the plan does not count -- e.g.
        # a conditional finalize -- is skipped instead of shifting the rest)
        want = [kernel_kind(f.launch_info(which, i)[0]) for i in range(n)]
        optional = ["skipped when" in f.launch_info(which, i)[0] for i in range(n)]
        picked, j = [], len(ks) - 1
        for _ in range(K):
            step_k = []
            for i in reversed(range(n)):
                if optional[i] and (j < 0 or not any(frag in ks[j].name for frag in want[i])):
                    step_k.append(None)  # e.g. a cast skipped because the input came as bf16
                    continue
                while j >= 0 and not any(frag in ks[j].name for frag in want[i]):
                    j -= 1
                if j < 0:
                    raise RuntimeError(f"CUPTI kernels do not match the plan (launch {i}: {want[i]})")
                step_k.append(ks[j])
                j -= 1
            picked = list(reversed(step_k)) + picked
        ks = picked
        if len(ks) == K * n:
            dur = [[0.0] * K for _ in range(n)]
            exc = [[0.0] * K for _ in range(n)]
            parts = [0] * n
            names = [""] * n
            last_end = None
            for j, e in enumerate(ks):
                k, i = divmod(j, n)
                if e is None:
                    names[i] = "(not launched)"
                    continue
                s0, e0 = e.start, e.start + e.dur
                dur[i][k] = e.dur * 1e-6
                parts[i] = max(parts[i], e.parts)
                exc[i][k] = max(0, e0 - (s0 if last_end is None else max(s0, last_end))) * 1e-6
                last_end = e0 if last_end is None else max(last_end, e0)
                names[i] = e.name
            out = []
            for i in range(n):
                desc, flops, nbytes = f.launch_info(which, i)
                out.append({"desc": desc, "kernel": names[i][:60], "ms": statistics.mean(dur[i]),
                            "excl_ms": statistics.mean(exc[i]), "flops": flops, "bytes": nbytes, "timing": "cupti",
                            "kernels": parts[i]})
    except Exception as ex:  # noqa: BLE001
        out = None
        why = repr(ex)[:200]
    if out is not None:
        return out
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(K)]
    for row in evs:
        for e in row:
            e.record()  # create the events
    torch.cuda.synchronize(dev)
    for k in range(K):
        f.set_launch_events(which, evs[k])
        step()
    f.set_launch_events(which, None)
    torch.cuda.synchronize(dev)
    out = []
    for i in range(n):
        desc, flops, nbytes = f.launch_info(which, i)
        ms = statistics.mean(evs[k][i].elapsed_time(evs[k][i + 1]) for k in range(K))
        out.append({"desc": desc, "ms": ms, "excl_ms": ms, "flops": flops, "bytes": nbytes, "timing": "events",
                    "cupti_failed": why})
    return out


def launched(kb):
    """Kernels a step really launches: the plan's launches minus the optional
    ones CUPTI saw skipped (a bf16 cast of bf16 input, a K-split sum step the
    GEMM made redundant by adding into an f32 home), counting both kernels of
    a hybrid GEMM launch."""
    return sum(r.get("kernels", 1) for r in kb if r.get("kernel") != "(not launched)")


def kernel_kind(desc):
    """Kernel-name fragments a plan launch with this description runs as."""
    if desc.startswith("gemm tcgen05"):
        return ("gemm_tc_kernel",)
    if desc.startswith("gemm simt"):
        return ("gemm_simt_kernel",)
    if desc.startswith("finalize"):
        return ("finalize_kernel",)
    if desc.startswith("pack"):
        return ("pack_bf16_kernel",)
    if desc.startswith("cast"):
        return ("cast_bf16_kernel",)
    return ("ew2d_kernel", "ew_kernel", "ew_tma_kernel")


# kernel-name fragments of this library's kernels (ahead-of-time and NVRTC)
OWN_KERNELS = ("gemm_tc_kernel", "gemm_simt_kernel", "ew_kernel", "ew2d_kernel", "ew_tma_kernel",
               "finalize_kernel", "cast_bf16_kernel", "pack_bf16_kernel")


def gemm_roofline(kb, pk, region_s, clocks=None):
    """Tensor roofline of a step's GEMMs.  `achieved` is the DOMINANT kernel's
    algorithmic FLOP (2*M*N*K summed over K segments) / its mean CUPTI
    duration.  Peak: the measured burst bf16 figure when the timed region
    lasted under 2 s (a kernel timed inside a short step), else the sustained
    one (MEASURED_PEAKS.json, measured power-capped); both fractions are
    reported, and the clocks beside them (a power-capped run shows a lower
    burst fraction rather than switching denominators: the sustained figure,
    measured at 1297 MHz, would put a 1500 MHz run above 1).  The GEMM class
    (all tcgen05/SIMT dots) is reported from exclusive times."""
    gemm = [r for r in kb if r["flops"] > 0]
    if not gemm:
        return None
    top = max(gemm, key=lambda r: r["ms"])
    burst, sus = pk["bf16_tflops"], pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    peak, kind = (burst, "burst") if region_s < 2.0 else (sus, "sustained")
    ach = top["flops"] / (top["ms"] * 1e-3) / 1e12
    g_ms = sum(r["excl_ms"] for r in gemm)
    g_fl = sum(r["flops"] for r in gemm)
    cls = g_fl / (g_ms * 1e-3) / 1e12 if g_ms else 0.0
    busy = sum(r["excl_ms"] for r in kb)
    return {"bound": "tensor", "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(ach / peak, 4), "traffic": None, "kernel": top["desc"][:100],
            "kernel_ms": round(top["ms"], 4), "kernel_flops": top["flops"], "timing": top["timing"],
            "peak_kind": f"{kind} bf16 ({pk['source']})", "frac_of_burst": round(ach / burst, 4),
            "frac_of_sustained": round(ach / sus, 4),
            "gemm_class": {"tflops": round(cls, 1), "frac_of_burst": round(cls / burst, 4),
                           "share_of_step": round(g_ms / busy, 4) if busy else None, "launches": len(gemm)}}


# -------------------------------------------------------- cpu baseline
def oracle_threads():
    n = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(n)
    except Exception:
        pass
    return n


def blas_info():
    """numpy version and the BLAS library / threads the oracle's dots ran on."""
    import numpy as np
    info = {"numpy": np.__version__}
    try:
        from threadpoolctl import threadpool_info
        blas = [p for p in threadpool_info() if p.get("user_api") == "blas"]
        if blas:
            info["blas"] = f"{blas[0].get('internal_api')} {blas[0].get('version')} ({blas[0].get('num_threads')} threads)"
    except Exception:  # noqa: BLE001
        pass
    return info


def cpu_baseline_mlp(w, rows: int):
    """The oracle (plain float64 numpy interpreter + reverse sweep) timed on
    `rows` rows of the same workload with full-size weights."""
    import numpy as np
    import oracle
    import workloads as W
    cores = oracle_threads()
    ws = W.c1(rows) if w.cfg == 1 else W.c3(rows, global_batch=w.global_batch, layers=w.layers)
    m = oracle.parse(ws.text)
    ins = [x.astype(np.float64) for x in ws.inputs()] + [np.float64(w.seed())]
    reps, t0 = 0, time.perf_counter()
    while True:  # passes over the same rows until >= 10 s of CPU work (bounded sample, ④)
        oracle.run(m, ws.grad, ins)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= 10.0:
            break
    out = {"value": rows * reps / dt, "unit": "samples/s", "cores": cores, "kind": "oracle",
           "sample": f"{rows} rows of {w.name} (full {len(w.layers)}-layer weights), {reps} fwd+adjoint pass(es), "
                     f"float64 numpy ({dt:.2f} s)", **blas_info()}
    try:  # one pass on one BLAS thread (the 1-thread time beside the all-core one)
        from threadpoolctl import threadpool_limits
        with threadpool_limits(1):
            t0 = time.perf_counter()
            oracle.run(m, ws.grad, ins)
            out["one_thread"] = round(rows / (time.perf_counter() - t0), 2)
    except Exception:  # noqa: BLE001
        pass
    return out


def cpu_baseline_chain(rows: int, C: int = 16384):
    import numpy as np
    import oracle
    import workloads as W
    cores = oracle_threads()
    w = W.c2(rows, C)
    m = oracle.parse(w.text)
    ins = [x.astype(np.float64) for x in w.inputs()]
    g = w.seed().astype(np.float64)
    t0 = time.perf_counter()
    oracle.run(m, w.fn, ins)
    oracle.run(m, w.grad, ins + [g])
    dt = time.perf_counter() - t0
    nbytes = rows * C * (12 + 16)
    return {"value": nbytes / dt / 1e9, "unit": "GB/s (algorithmic)", "cores": cores, "kind": "oracle",
            "sample": f"{rows}x{C} rows of c2, fwd + fwd-adjoint, float64 numpy ({dt:.2f} s)"}


# ----------------------------------------------------------------- main
def ncu_traffic(name):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    of the workload's dominant kernel from the committed ncu --set full
    capture (profiles/ncu_traffic.json), or None."""
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(prof)).get(name)
    except Exception:  # noqa: BLE001
        return None


def bench_chain(dev, K, W_):
    """config 2: y = tanh(x*w + b)*m and its adjoint on [16384, 16384] f32."""
    import torch
    import numpy as np
    import paper_1711_03016_b200 as P
    import workloads as WL
    w = WL.c2()
    f = P.Function(w.text, w.fn, w.grad)
    ins = [to_dev(x, dev) for x in w.inputs()]
    seed = to_dev(w.seed(), dev)
    (y,) = f._outputs(0, dev, None)
    gouts = f._outputs(1, dev, None)
    ws0, ws1 = f._workspace(0, dev), f._workspace(1, dev)
    fwd = lambda: f.run(ins, outputs=[y], workspace=ws0)
    adj = lambda: f.grad_run(ins, seed=seed, outputs=gouts, workspace=ws1)
    for _ in range(W_):
        fwd()
        adj()
    ms_f = time_steps(fwd, K, dev, 1)
    ms_a = time_steps(adj, K, dev, 1)
    n = 16384 * 16384
    bf, ba = 12.0 * n, 16.0 * n
    kb = kernel_breakdown(f, 1, adj, min(K, 5), dev)
    main = max(kb, key=lambda r: r["ms"])
    pk = peaks()
    hb = pk["hbm_gbs"]
    gbs_k = ba / (main["ms"] * 1e-3) / 1e9
    gbs_f, gbs_a = bf / (ms_f * 1e-3) / 1e9, ba / (ms_a * 1e-3) / 1e9
    detail = {"fwd_adj_kernels": [dict(r, desc=r["desc"][:100]) for r in kb]}
    return {"workload": "c2_chain [16384,16384] f32", "fwd_ms": round(ms_f, 4), "fwd_gbs": round(gbs_f, 1),
            "fwd_frac": round(gbs_f / hb, 4), "fwd_adj_ms": round(ms_a, 4), "fwd_adj_gbs": round(gbs_a, 1),
            "fwd_adj_frac": round(gbs_a / hb, 4),
            "roofline": {"bound": "hbm", "achieved": round(gbs_k, 1), "peak": hb, "unit": "GB/s",
                         "frac": round(gbs_k / hb, 4),
                         "traffic": (ncu_traffic("c2_chain") or {}).get("traffic_bytes"),
                         "kernel": main["desc"][:80], "algorithmic_bytes": ba, "timing": main["timing"]},
            "launches_fwd_adj": f.num_launches(1)}, detail


def bench_grad_leg(w, small, dev, K, W_, bf16_args, cpu_rows):
    """One gradient step of a NEXT-row workload (rnn: linear algebra fusion;
    mlp_hvp: a second-order gradient) through dlvm_grad_run: samples/s,
    algorithmic TFLOP/s of its GEMMs against the tensor roofline, and the
    oracle on a bounded row sample of the same program (`small(rows)`)."""
    import numpy as np
    import torch
    import oracle
    import paper_1711_03016_b200 as P
    f = P.Function(w.text, w.fn, w.grad, dot_precision=w.dot_precision)
    ins = [to_dev(x, dev, a.name in bf16_args) for x, a in zip(w.inputs(), w.args)]
    sd = w.seed()
    seed = to_dev(np.asarray(sd, dtype=np.float32), dev) if sd is not None else None
    outs = f._outputs(1, dev, None)
    ws = f._workspace(1, dev)
    step = lambda: f.grad_run(ins, seed=seed, outputs=outs, workspace=ws)
    for _ in range(W_):
        step()
    ms = time_steps(step, K, dev, 1)
    kb = kernel_breakdown(f, 1, step, min(K, 5), dev)
    flops = sum(r["flops"] for r in kb)
    pk = peaks()
    out = {"workload": w.name, "value": round(w.global_batch / (ms * 1e-3), 1), "unit": "samples/s",
           "ms_per_step": round(ms, 4), "step_tflops": round(flops / (ms * 1e-3) / 1e12, 1),
           "step_frac_of_burst": round(flops / (ms * 1e-3) / 1e12 / pk["bf16_tflops"], 4),
           "launches": launched(kb), "roofline": gemm_roofline(kb, pk, ms * K * 1e-3)}
    detail = [dict(r, desc=r["desc"][:110]) for r in kb]
    try:
        cores = oracle_threads()
        ws_ = small(cpu_rows)
        m = oracle.parse(ws_.text)
        args = [x.astype(np.float64) for x in ws_.inputs()]
        sd = ws_.seed()
        if sd is not None:
            args.append(np.asarray(sd, dtype=np.float64))
        t0 = time.perf_counter()
        oracle.run(m, ws_.grad, args)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": cpu_rows / dt, "unit": "samples/s", "cores": cores, "kind": "oracle",
                               "sample": f"{cpu_rows} rows of {w.name} (full-size weights), float64 numpy ({dt:.2f} s)"}
    except Exception as ex:  # noqa: BLE001
        out["cpu_baseline"] = {"error": repr(ex)}
    return out, detail


def spawn_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: re-run this command as N ranks (one
    process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _pick(d, keys):
    return {k: d[k] for k in keys if d is not None and k in d}


def compact_line(out):
    """The one JSON line: every contract key, and of each sub-measurement
    only its headline numbers (the full records go to the detail file), so
    the line stays short enough for the driver's stdout tail."""
    line = _pick(out, ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "step_ms",
                       "higher_is_better",
                       "scaling", "vs_baseline", "dtype", "data", "config", "step_tflops", "gpu_launches", "clocks"])
    line["config"] = _pick(out["config"], ["workload", "global_batch", "per_rank_batch", "parallelism", "l2",
                                           "cuda_graph", "step", "gradient_reduction"])
    r = out.get("roofline")
    if r:
        line["roofline"] = _pick(r, ["bound", "achieved", "peak", "unit", "frac", "traffic", "kernel_ms", "timing",
                                     "frac_of_sustained"])
        line["roofline"]["kernel"] = r["kernel"][:60]
        line["roofline"]["peak_kind"] = r["peak_kind"].split(" (")[0]
        line["roofline"]["gemm_class"] = _pick(r["gemm_class"], ["tflops", "frac_of_burst", "share_of_step"])
    if "e2e" in out:
        e = out["e2e"]
        line["e2e"] = _pick(e, ["value", "unit", "ms_per_step", "h2d_bytes_per_step", "d2h_bytes_per_step",
                                "x_host_dtype"])
        if "f32_inputs" in e:
            line["e2e"]["f32_inputs"] = _pick(e["f32_inputs"], ["value", "ms_per_step", "h2d_bytes_per_step"])
    if "cpu_baseline" in out:
        line["cpu_baseline"] = out["cpu_baseline"]
    if "fused_elementwise" in out:
        ew = out["fused_elementwise"]
        line["fused_elementwise"] = _pick(ew, ["fwd_gbs", "fwd_frac", "fwd_adj_gbs", "fwd_adj_frac"])
        line["fused_elementwise"]["roofline"] = _pick(ew["roofline"], ["bound", "achieved", "peak", "unit", "frac",
                                                                        "traffic", "timing"])
        line["fused_elementwise"]["cpu_gbs"] = (ew.get("cpu_baseline") or {}).get("value")
    legs = dict(out.get("other_configs", {}))
    legs.update(out.get("next_rows", {}))
    for name, leg in legs.items():
        c = _pick(leg, ["value", "ms_per_step", "step_tflops", "step_frac_of_burst"])
        if leg.get("roofline"):
            c["gemm_frac_of_burst"] = leg["roofline"]["gemm_class"]["frac_of_burst"]
            c["top_kernel_frac"] = leg["roofline"]["frac"]
        c["cpu_samples_s"] = (leg.get("cpu_baseline") or {}).get("value")
        line.setdefault("other_configs" if name in out.get("other_configs", {}) else "next_rows", {})[name] = c
    return line


def write_detail(args, detail):
    """Per-kernel lists and the other long records go to a file, so the one
    JSON line stays short (`--detail PATH`; default gpurun_out/ when it
    exists)."""
    path = args.detail
    if path is None and os.path.isdir(os.path.join(ROOT, "gpurun_out")):
        path = os.path.join(ROOT, "gpurun_out", f"bench_detail_{args.workload}_n{detail['n_gpus']}.json")
    if path:
        with open(path, "w") as fh:
            json.dump(detail, fh, indent=1)
    return path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c4", choices=["c4", "c3", "c1", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-elementwise", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-e2e-f32", action="store_true", help="skip the e2e variant with f32 host inputs")
    ap.add_argument("--no-next", action="store_true", help="skip the rnn / mlp_hvp legs (SURVEY §8(f) rows)")
    ap.add_argument("--no-configs", action="store_true", help="skip the c3 leg (BASELINE config 3, batch 1024)")
    ap.add_argument("--cpu-rows", type=int, default=None)
    ap.add_argument("--detail", default=None, help="write per-kernel detail JSON here")
    ap.add_argument("--dp", default="nccl", choices=["nccl", "fused"],
                    help="gradient reduction: bucketed NCCL all-reduce, or fused into the gradient kernels "
                         "(DLVM_F32_ADD into the owners' symmetric memory, dp.FusedReduceStep)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as a CUDA graph (auto: on for the launch-bound c1)")
    args = ap.parse_args()
    W_ = max(3, args.warmup)
    K = args.steps
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    import workloads as WL

    def make_workload():
        if args.workload == "c4":
            return WL.c4(world)
        if args.workload == "c3":
            return WL.c3()
        if args.workload == "c1":
            return WL.c1()
        return WL.c5(131072 // max(world, 1), 131072)

    if args.impl == "reference":
        if rank != 0:
            return
        w = make_workload()
        rows = 64 if args.workload in ("c4", "c3") else (32 if args.workload == "c1" else 16)
        import numpy as np
        import oracle
        cores = oracle_threads()
        ws = WL.c3(rows, global_batch=w.global_batch, layers=w.layers) if args.workload != "c1" else WL.c1(rows)
        m = oracle.parse(ws.text)
        ins = [x.astype(np.float64) for x in ws.inputs()] + [np.float64(w.seed())]
        for _ in range(W_):
            oracle.run(m, ws.grad, ins)
        t0 = time.perf_counter()
        for _ in range(K):
            oracle.run(m, ws.grad, ins)
        dt = (time.perf_counter() - t0) / K
        v = rows / dt
        cb = {"value": v, "unit": "samples/s", "cores": cores, "kind": "oracle",
              "sample": f"{rows} rows of {w.name} per step, float64 numpy"}
        print(json.dumps({"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus, "steps": K,
                          "warmup": W_, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                          "config": {"workload": w.name, "global_batch": w.global_batch, "sample_rows": rows,
                                     "parallelism": f"dp{args.gpus}"},
                          "cpu_baseline": cb,
                          "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1711_03016_b200 as P
    from paper_1711_03016_b200.dp import DataParallelStep

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.dp == "fused":
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        else:
            dist.init_process_group("nccl", device_id=dev)
        assert dist.get_world_size() == args.gpus, (dist.get_world_size(), args.gpus)
    pk = peaks()
    w = make_workload()
    f, dev_in, seed, host, n_grads = mlp_setup(w, dev, rank)
    if args.dp == "fused":
        from paper_1711_03016_b200.dp import FusedReduceStep
        dps = FusedReduceStep(f, n_grads, dev)
        dps.grads = type("G", (), {"views": dps.views})()
    else:
        dps = DataParallelStep(f, n_grads, dev, world_size=world)
        for e in dps.events:
            e.record()
    train_step = lambda inp: dps.step(inp, seed)
    step = lambda: train_step(dev_in)
    sgd_info = None
    if args.workload == "c5" and args.dp == "fused":
        # training step with the fused reduction and the sharded update:
        # owners update their fp32 masters and all-gather the operand copies
        from paper_1711_03016_b200.dp import ShardedSGD
        dps.gather = False
        copies = [a.name.startswith("w") for a in w.args[1:-1]]
        upd = ShardedSGD(dps, host[1:-1], copies, 1e-3, WL.sgd_ir)
        for j in range(len(copies)):
            dev_in[1 + j] = upd.operands[j]

        def train_step(inp):
            outs = dps.step(inp, seed)
            upd.step()
            return outs

        step = lambda: train_step(dev_in)
        sgd_info = {"launches": upd.sgd.num_launches(0) if upd.sgd else 0,
                    "params": int(sum(np.prod(a.shape) for a in w.args[1:-1]))}
    elif args.workload == "c5":
        # full training step (config 5): fwd + adjoint, gradient all-reduce, and
        # the SGD update W <- W - lr*G (an IR function through the same C ABI)
        # writing the fp32 master and the bf16 copy the next step's dots read
        shapes = [a.shape for a in w.args[1:-1]]
        copies = [a.name.startswith("w") for a in w.args[1:-1]]
        sgd = P.Function(WL.sgd_ir(shapes, 1e-3, copies), "sgd", None)
        masters = [torch.from_numpy(x).to(dev) for x in host[1:-1]]
        for j, a in enumerate(w.args[1:-1]):
            if not copies[j]:
                dev_in[1 + j] = masters[j]  # biases: the fp32 master is the grad input
        sgd_in, sgd_out = [], []
        for j, a in enumerate(w.args[1:-1]):
            sgd_in += [masters[j], dps.grads.views[j]]
            sgd_out.append(masters[j])
            if copies[j]:
                sgd_out.append(dev_in[1 + j])  # bf16 operand copy, updated in place
        sgd_ws = sgd._workspace(0, dev)

        def train_step(inp):
            outs = dps.step(inp, seed)
            sgd.run(sgd_in, outputs=sgd_out, workspace=sgd_ws)
            return outs

        step = lambda: train_step(dev_in)

        sgd_info = {"launches": sgd.num_launches(0), "params": int(sum(np.prod(x) for x in shapes))}
    for _ in range(W_):
        step()
    torch.cuda.synchronize(dev)
    eager_step = step
    use_graph = args.graph == "on" or (args.graph == "auto" and args.workload == "c1")
    if use_graph and world == 1:
        # dlvm_grad_run neither allocates nor synchronises, so the whole step
        # (all launches + gradient-ready events) is capturable
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            eager_step()
        step = graph.replay
        for _ in range(W_):
            step()
        torch.cuda.synchronize(dev)
    else:
        use_graph = False
    with ClockSampler(local) as clk:
        t0 = time.time()
        step_stats = {}
        ms = time_steps(step, K, dev, world, stats=step_stats)
        clk.window = (t0, time.time())
    clocks = clk.summary()
    value = w.global_batch / (ms * 1e-3)
    # per-kernel breakdown: a separate short pass under CUPTI activity tracing
    # (the timed region above runs without any profiler)
    kb = kernel_breakdown(f, 1, eager_step, min(K, 5), dev)
    roof = gemm_roofline(kb, pk, ms * K * 1e-3, clocks)
    tr = ncu_traffic(w.name)
    if tr and roof:
        # the capture of the kernel the roofline names (its %value in the
        # plan description), else the workload's dominant-kernel capture
        import re
        m = re.search(r"(%\w+)", roof["kernel"])
        per = tr.get("kernels", {}).get(m.group(1)) if m else None
        if per:
            roof["traffic"] = per["traffic_bytes"]
            roof["traffic_kernel"] = m.group(1)
            roof["traffic_source"] = tr["kernels_source"]
        else:
            roof["traffic"] = tr["traffic_bytes"]
            roof["traffic_kernel"] = tr["kernel"]
            roof["traffic_source"] = tr["source"]
    step_flops = sum(r["flops"] for r in kb)
    launches = (launched(kb) + (sgd_info["launches"] if sgd_info else 0)) * K
    detail = {"n_gpus": world, "workload": w.name,
              "kernels": [{"desc": r["desc"][:120], "kernel": r.get("kernel"), "ms": round(r["ms"], 4),
                           "excl_ms": round(r["excl_ms"], 4), "flops": r["flops"], "bytes": r["bytes"],
                           "timing": r["timing"], "kernels": r.get("kernels", 1)} for r in kb]}

    def e2e_leg(f32_inputs: bool):
        """End to end through the public API: every step copies its own batch
        (x, t) from pinned host memory and reads the loss back.  Two device
        copies of the batch arguments alternate: step k+1's upload runs on a
        copy stream while step k computes.  `f32_inputs`: x is uploaded in
        the IR's f32 type (the library casts it for the bf16 dots) instead of
        the bf16 storage form dlvm.h allows."""
        xi = [i for i, a in enumerate(w.args) if a.batched]
        pinned = []
        bufs = [list(dev_in), list(dev_in)]
        for i in xi:
            t = torch.from_numpy(host[i])
            if dev_in[i].dtype == torch.bfloat16 and not f32_inputs:
                t = t.to(torch.bfloat16)
            elif dev_in[i].dtype == torch.bool:
                t = t != 0
            pinned.append(t.pin_memory())
            bufs[0][i] = torch.empty(t.shape, dtype=t.dtype, device=dev)
            bufs[1][i] = torch.empty(t.shape, dtype=t.dtype, device=dev)
        loss_h = torch.empty((), dtype=torch.float32).pin_memory()
        h2d = sum(p.numel() * p.element_size() for p in pinned)
        copy_st = torch.cuda.Stream(device=dev)
        main_st = torch.cuda.current_stream(dev)
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        state = {"k": 0}

        def upload(slot):
            with torch.cuda.stream(copy_st):
                copy_st.wait_event(free[slot])
                for i, p in zip(xi, pinned):
                    bufs[slot][i].copy_(p, non_blocking=True)
                ready[slot].record(copy_st)

        for e in free:
            e.record(main_st)

        def e2e_step():
            k = state["k"]
            slot = k % 2
            if k == 0:
                upload(slot)
            upload(1 - slot)  # next step's batch, overlapping this step's compute
            main_st.wait_event(ready[slot])
            outs = train_step(bufs[slot])
            free[slot].record(main_st)
            loss_h.copy_(outs[-1], non_blocking=True)
            state["k"] = k + 1

        for _ in range(2):
            e2e_step()
        ms_e2e = time_steps(e2e_step, max(3, K // 2), dev, world)
        torch.cuda.synchronize(dev)
        del bufs
        return {"value": round(w.global_batch / (ms_e2e * 1e-3), 1), "unit": "samples/s",
                "ms_per_step": round(ms_e2e, 4), "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": 4 * world,
                "x_host_dtype": "f32" if f32_inputs else str(dev_in[0].dtype).replace("torch.", "")}

    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(False)
        e2e["api"] = "Function.grad_run (dlvm_grad_run) + DataParallelStep; batch upload of step k+1 overlaps step k"
        if not args.no_e2e_f32 and w.dot_precision == "bf16":
            e2e["f32_inputs"] = e2e_leg(True)
    out = {"metric": METRIC, "value": round(value, 1), "unit": "samples/s", "n_gpus": world, "steps": K,
           "warmup": W_, "ms_per_step": round(ms, 4), "step_ms": step_stats, "higher_is_better": True,
           "scaling": "strong",
           "vs_baseline": None, "dtype": "bf16" if w.dot_precision == "bf16" else "f32",
           "data": "synthetic (seeded PCG64 per workloads.py; Glorot weights)",
           "config": {"workload": w.name, "global_batch": w.global_batch, "per_rank_batch": w.batch,
                      "layers": [list(l) for l in w.layers], "parallelism": f"dp{world}",
                      "dot_precision": "bf16 operands, fp32 accumulate (tcgen05)" if w.dot_precision == "bf16"
                      else "fp32 operands, FFMA (SIMT)",
                      "gradient_reduction": "fused into the gradient kernels (DLVM_F32_ADD into owners' peer memory)"
                      if args.dp == "fused" else "bucketed NCCL all-reduce on a comm stream",
                      "l2": ("inputs larger than L2 (x is %d MiB per rank)" % (w.batch * w.layers[0][0] * 2 >> 20))
                      if w.cfg != 1 else "L2-resident (whole c1 working set < 1 MiB; latency-bound config)",
                      "cuda_graph": use_graph},
           "step_tflops": round(step_flops / (ms * 1e-3) / 1e12, 1),
           "roofline": roof, "gpu_launches": launches, "clocks": clocks}
    if e2e:
        out["e2e"] = e2e
    if sgd_info:
        out["config"]["step"] = ("fwd+adjoint + fused gradient reduction + sharded SGD update (lr 1e-3) + all-gather "
                                 "of %d params" if args.dp == "fused" else
                                 "fwd+adjoint + gradient all-reduce + SGD update (lr 1e-3) of %d params") % sgd_info["params"]
    if rank == 0 and world == 1:
        try:
            out["cpu_baseline"] = cpu_baseline_mlp(w, args.cpu_rows or (32 if w.cfg == 1 else 128))
        except Exception as ex:  # noqa: BLE001
            out["cpu_baseline"] = {"error": repr(ex)}
        if not args.no_elementwise:
            ew, ew_detail = bench_chain(dev, K, W_)
            out["fused_elementwise"] = ew
            detail["fused_elementwise"] = ew_detail
            out["gpu_launches"] += (1 + ew["launches_fwd_adj"]) * K
            try:
                ew["cpu_baseline"] = cpu_baseline_chain(256)
            except Exception as ex:  # noqa: BLE001
                ew["cpu_baseline"] = {"error": repr(ex)}
        if not args.no_configs and args.workload == "c4":
            # BASELINE config 3 (the same MLP at batch 1024; target >= 975.5 TFLOP/s,
            # BASELINE.md §3) through dlvm_grad_run, x and W as bf16 storage
            c3, detail["c3"] = bench_grad_leg(WL.c3(), lambda r: WL.c3(r), dev, K, W_, {"x", "w1", "w2", "w3"}, 64)
            out["gpu_launches"] += c3["launches"] * K
            out["other_configs"] = {"c3": c3}
        if not args.no_next:
            legs = {}
            rnn = WL.rnn()
            legs["rnn"], detail["rnn"] = bench_grad_leg(rnn, lambda r: WL.rnn(8, r, 2048, 2048), dev, K, W_,
                                                        {"W", "U", "h0"} | {f"x{t}" for t in range(1, 9)}, 16)
            hv = WL.mlp_hvp()
            legs["mlp_hvp"], detail["mlp_hvp"] = bench_grad_leg(hv, lambda r: WL.mlp_hvp(r), dev, K, W_,
                                                                {"x", "W1", "W2"}, 16)
            for v in legs.values():
                out["gpu_launches"] += v["launches"] * K
            out["next_rows"] = legs
    if rank == 0:
        detail["line_full"] = out
        dp_ = write_detail(args, detail)
        line = compact_line(out)
        if dp_:
            line["detail_file"] = os.path.relpath(dp_, ROOT)
        print(json.dumps(line))
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
