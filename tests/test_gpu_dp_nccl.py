"""Data parallelism on >= 2 GPUs over NCCL: each rank runs
DataParallelStep.step -- dlvm_grad_run on its row shard, gradient-ready
events, bucketed all-reduce on the comm stream -- and the summed gradients
must equal the oracle's gradient of the GLOBAL batch (F15).  Skipped when
fewer than 2 GPUs are visible (the round's GPU boxes have one)."""

import os
import socket

import numpy as np
import pytest

import oracle
import workloads as W
from helpers import assert_f32_parity, assert_normwise, oracle_grad_module, term_bound

pytestmark = pytest.mark.gpu

GB = 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(prec, world):
    """The c3 program shape at reduced width: tanh layers under the fp32 dot
    policy (SIMT GEMMs, A17 bounds), ReLU layers under bf16 (tcgen05, A18')."""
    act = "tanh" if prec == "f32" else "relu"
    return W.c3(GB // world, global_batch=GB, layers=[(256, 512, act), (512, 512, act), (512, 128, None)])


def _worker(rank, world, port, prec, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import paper_1711_03016_b200 as P
    from paper_1711_03016_b200.dp import DataParallelStep
    w = _case(prec, world)
    f = P.Function(w.text, w.fn, w.grad, dot_precision=prec)
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs(row_offset=rank * w.batch)]
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    dps = DataParallelStep(f, 2 * len(w.layers), dev, world_size=world)
    outs = dps.step(ins, seed)
    torch.cuda.synchronize(dev)
    if rank == 0:
        out.put([o.double().cpu().numpy() for o in outs])
    dist.destroy_process_group()


@pytest.mark.parametrize("prec", ["f32", "bf16"])
def test_data_parallel_step_nccl_two_ranks(prec):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, prec, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = _case(prec, 1)
    m = oracle.parse(w.text)
    args = [x.astype(np.float64) for x in w.inputs()] + [np.float64(w.seed())]
    if prec == "f32":
        ref = oracle.run(m, w.grad, args)
        bounds = term_bound(oracle_grad_module(m, w.grad), w.grad, args)
        for k, (g, r, b) in enumerate(zip(got, ref, bounds)):
            # the kept loss is this rank's shard loss (not all-reduced)
            if k < len(got) - 1:
                assert_f32_parity(g, r, b, what=f"dp grad out{k}")
    else:
        ref = oracle.run(m, w.grad, args, dot_policy="bf16")
        for k, (g, r) in enumerate(zip(got[:-1], ref[:-1])):
            assert_normwise(g, r, what=f"dp bf16 grad out{k}")
