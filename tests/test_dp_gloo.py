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


# --- DataParallelStep itself (bucket order, event gating) on gloo -----------

class _LogStreams:
    """CPU stand-in for dp.CudaStreams that logs every stream operation."""

    def __init__(self, log):
        self.log = log
        self.k = 0

    def new_event(self):
        self.k += 1
        return ("event", self.k - 1)

    def new_stream(self):
        return "comm"

    def current(self):
        return "compute"

    def use(self, stream):
        import contextlib
        log = self.log

        @contextlib.contextmanager
        def ctx():
            log.append(("enter", stream))
            yield
            log.append(("exit", stream))
        return ctx()

    def wait_event(self, stream, event):
        self.log.append(("wait", stream, event[1]))

    def wait_stream(self, stream, other):
        self.log.append(("wait_stream", stream, other))

    def handle(self, stream):
        return stream


class _OracleGradFn:
    """Stand-in for a gradient handle on CPU: grad_run computes this rank's
    shard gradients with the oracle and writes them into the caller's
    outputs in the order the planner finalises them (last layer first),
    "recording" gradient g's ready event right after g is written."""

    def __init__(self, w, log):
        self.w, self.log = w, log
        self.m = oracle.parse(w.text)

    def signature(self, which):
        g = self.m.functions[self.w.grad]
        return None, [(tuple(t.shape), t.dtype) for t in g.result_types]

    def grad_run(self, inputs, seed, outputs, stream, events):
        self.log.append(("grad_run", stream))
        res = oracle.run(self.m, self.w.grad, list(inputs) + [np.float64(seed)])
        n = len(res) - 1
        order = []
        for l in reversed(range(n // 2)):
            order += [2 * l, 2 * l + 1]
        for g in order + [n]:
            outputs[g].copy_(torch.from_numpy(np.asarray(res[g], dtype=np.float64)).reshape(outputs[g].shape))
            if g < n and events is not None:
                self.log.append(("ready", events[g][1]))


def _dps_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_03016_b200.dp import DataParallelStep
    w = W.c3(GB // world, global_batch=GB, layers=LAYERS)
    log = []
    fn = _OracleGradFn(w, log)
    n_grads = 2 * len(w.layers)
    dps = DataParallelStep(fn, n_grads, "cpu", world_size=world, streams=_LogStreams(log),
                           grads_dtype=torch.float64)
    ins = [x.astype(np.float64) for x in w.inputs(row_offset=rank * w.batch)]
    outs = dps.step(ins, 1.0 / GB)
    if rank == 0:
        out.put(([o.clone().numpy() for o in outs[:n_grads]], log, dps.buckets))
    dist.destroy_process_group()


def test_data_parallel_step_two_ranks_bucket_order_and_event_gating():
    """DataParallelStep.step on gloo (world size 2) with the oracle standing in
    for dlvm_grad_run: the all-reduced gradients equal the global-batch
    gradient (F15); buckets are issued on the comm stream in reverse layer
    order; each bucket's all-reduce is preceded, inside the comm stream, by
    waits on exactly its gradients' ready events, each recorded before; the
    compute stream finally waits for the comm stream."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dps_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, log, buckets = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.c3(GB, layers=LAYERS)
    m = oracle.parse(w.text)
    ref = oracle.run(m, w.grad, [x.astype(np.float64) for x in w.inputs()] + [np.float64(1.0 / GB)])[:-1]
    for g, r in zip(got, ref):
        np.testing.assert_allclose(g, r, rtol=1e-12, atol=1e-15)
    assert log[0] == ("grad_run", "compute")
    ready_at = {e[1]: i for i, e in enumerate(log) if e[0] == "ready"}
    issued = []
    i = 0
    while i < len(log):
        if log[i] == ("enter", "comm"):
            j = log.index(("exit", "comm"), i)
            waits = [e[2] for e in log[i + 1:j] if e[0] == "wait"]
            assert all(e[1] == "comm" for e in log[i + 1:j] if e[0] == "wait")
            for g in waits:
                assert ready_at[g] < i  # the event was recorded before the comm stream waits on it
            issued.append(waits)
            i = j
        i += 1
    assert issued == [list(b) for b in reversed(buckets)]
    assert log[-1] == ("wait_stream", "compute", "comm")


def test_assign_owners_balanced_and_deterministic():
    from paper_1711_03016_b200.dp import assign_owners
    sizes = [4096 * 4096, 4096, 4096 * 4096, 4096, 4096 * 1000, 1000]
    assert assign_owners(sizes, 1) == [0] * 6
    o2 = assign_owners(sizes, 2)
    assert o2[0] != o2[2]  # the two big gradients on different ranks
    load = [sum(s for s, o in zip(sizes, o2) if o == r) for r in range(2)]
    assert max(load) - min(load) <= 4096 * 1000 + 4096 + 1000
    assert assign_owners(sizes, 8) == assign_owners(list(sizes), 8)
    assert sorted(set(assign_owners(sizes, 8))) == list(range(6))
