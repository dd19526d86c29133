"""Data-parallel host logic on CPU (gloo, world size 2): each rank computes
its batch shard's gradients (the oracle stands in for dlvm_grad_run, which
needs a GPU), writes them into the flat bucketed gradient buffer of
paper_1711_03016_b200.dp, and all-reduces the buckets in reverse layer
order.  The result must equal the global-batch gradient (F15: linearity of
the adjoint in the seed 1/B_global)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W

LAYERS = [(12, 10, "relu"), (10, 6, None)]
GB = 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_03016_b200.dp import GradBuffer, allreduce_buckets, layer_buckets
    w = W.c3(GB // world, global_batch=GB, layers=LAYERS)
    m = oracle.parse(w.text)
    ins = [x.astype(np.float64) for x in w.inputs(row_offset=rank * w.batch)]
    grads = oracle.run(m, w.grad, ins + [np.float64(1.0 / GB)])[:-1]
    buf = GradBuffer([g.shape for g in grads], "cpu", dtype=torch.float64)
    for v, g in zip(buf.views, grads):
        v.copy_(torch.from_numpy(g))
    buckets = layer_buckets(len(grads))
    works = allreduce_buckets(buf, buckets, order=list(reversed(range(len(buckets)))))
    for wk in works:
        wk.wait()
    if rank == 0:
        out.put([v.clone().numpy() for v in buf.views])
    dist.destroy_process_group()


def test_dp_two_ranks_equals_global_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.c3(GB, layers=LAYERS)
    m = oracle.parse(w.text)
    ref = oracle.run(m, w.grad, [x.astype(np.float64) for x in w.inputs()] + [np.float64(1.0 / GB)])[:-1]
    for g, r in zip(got, ref):
        np.testing.assert_allclose(g, r, rtol=1e-12, atol=1e-15)


def test_flat_layout_alignment_and_buckets():
    from paper_1711_03016_b200.dp import GradBuffer, flat_layout, layer_buckets
    offs, total = flat_layout([(4096, 4096), (1, 4096), (4096, 1000), (1, 1000)])
    assert all(o % 64 == 0 for o in offs)          # 256-byte aligned fp32 gradients
    assert total >= 4096 * 4096 + 4096 + 4096 * 1000 + 1000
    assert layer_buckets(6) == [[0, 1], [2, 3], [4, 5]]
    buf = GradBuffer([(3, 5), (1, 5), (5, 2), (1, 2)], "cpu")
    s = buf.bucket_slice([0, 1])
    assert s.data_ptr() == buf.views[0].data_ptr()
    assert s.numel() == buf.offsets[1] + 5
