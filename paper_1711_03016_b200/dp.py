"""Batch-sharded data parallelism (BASELINE.json north_star:
"forward plus adjoint is sharded along the batch dimension, with one NCCL
allreduce over NVLink of the parameter gradients").

Rank r owns rows [r*B/N, (r+1)*B/N) of the batch arguments; weights are
replicated.  Every forward op and every activation adjoint is row-local;
only the contractions over the batch (dW = H^T dZ, db = sum_rows dZ, the
loss) need combining.  With the seed 1/B_global the SUM all-reduce yields
the global-batch gradient (pin F15).

Gradients land in one flat fp32 buffer laid out per parameter; buckets are
contiguous runs of parameters (one layer's dW and db) all-reduced on a
communication stream as soon as dlvm_grad_run records the gradient-ready
event of the bucket's last gradient, so the all-reduce of layer L overlaps
the adjoint of layers L-1..1 (the planner emits the dW GEMMs in reverse
layer order)."""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple


def flat_layout(shapes: Sequence[Tuple[int, ...]], align: int = 64) -> Tuple[List[int], int]:
    """Element offsets of each gradient in the flat buffer (each 256-byte
    aligned, as the C ABI wants 16-byte-aligned outputs) and the total size."""
    offs, n = [], 0
    for s in shapes:
        offs.append(n)
        k = 1
        for d in s:
            k *= d
        n += (k + align - 1) // align * align
    return offs, n


def layer_buckets(n_grads: int, per_bucket: int = 2) -> List[List[int]]:
    """Buckets of consecutive gradients: (dW_l, db_l) pairs for MLPs."""
    return [list(range(i, min(i + per_bucket, n_grads))) for i in range(0, n_grads, per_bucket)]


class GradBuffer:
    """Flat gradient storage + per-gradient views (torch tensors)."""

    def __init__(self, shapes: Sequence[Tuple[int, ...]], device, dtype=None):
        import torch
        self.shapes = [tuple(s) for s in shapes]
        self.offsets, total = flat_layout(self.shapes)
        self.flat = torch.zeros(total, dtype=dtype or torch.float32, device=device)
        self.views = []
        for o, s in zip(self.offsets, self.shapes):
            k = 1
            for d in s:
                k *= d
            self.views.append(self.flat[o:o + k].view(s))

    def bucket_slice(self, bucket: Sequence[int]):
        lo = self.offsets[bucket[0]]
        last = bucket[-1]
        k = 1
        for d in self.shapes[last]:
            k *= d
        return self.flat[lo:self.offsets[last] + k]


class CudaStreams:
    """The stream/event operations DataParallelStep needs, on CUDA (the
    product configuration).  Tests on CPU substitute an object with the same
    methods to observe bucket order and event gating (tests/test_dp_gloo.py)."""

    def __init__(self, device):
        import torch
        self.torch = torch
        self.device = device

    def new_event(self):
        e = self.torch.cuda.Event()
        e.record()  # torch creates CUDA events lazily; the C ABI needs real handles
        return e

    def new_stream(self):
        return self.torch.cuda.Stream(device=self.device)

    def current(self):
        return self.torch.cuda.current_stream(self.device)

    def use(self, stream):
        return self.torch.cuda.stream(stream)

    def wait_event(self, stream, event):
        stream.wait_event(event)

    def wait_stream(self, stream, other):
        stream.wait_stream(other)

    def handle(self, stream):
        return stream.cuda_stream


def allreduce_buckets(buf: GradBuffer, buckets: Sequence[Sequence[int]], group=None, order=None,
                      comm_stream=None, ready_events=None, streams=None):
    """All-reduce (SUM) each bucket.  With `comm_stream` and `ready_events`
    (one event per gradient), bucket b is issued on the comm stream after
    waiting for the events of its gradients.  Returns the async work handles
    (the caller makes its stream wait on them)."""
    import torch.distributed as dist
    works = []
    seq = order if order is not None else range(len(buckets))
    for b in seq:
        bucket = buckets[b]
        if comm_stream is not None:
            if streams is None:
                streams = CudaStreams(None)
            with streams.use(comm_stream):
                if ready_events is not None:
                    for g in bucket:
                        streams.wait_event(comm_stream, ready_events[g])
                works.append(dist.all_reduce(buf.bucket_slice(bucket), op=dist.ReduceOp.SUM, group=group,
                                             async_op=True))
        else:
            works.append(dist.all_reduce(buf.bucket_slice(bucket), op=dist.ReduceOp.SUM, group=group,
                                         async_op=True))
    return works


class DataParallelStep:
    """One fwd+adjoint step of a gradient handle on this rank's batch shard,
    then the bucketed gradient all-reduce (NCCL), overlapped with the adjoint:
    dlvm_grad_run records gradient g's ready event on the compute stream as
    soon as g is final; bucket b's all-reduce is issued on a communication
    stream that first waits for the events of b's gradients, in reverse
    bucket order (the last layer's gradients are final first)."""

    def __init__(self, fn, n_grads: int, device, group=None, per_bucket: int = 2, world_size: int = 1,
                 streams=None, grads_dtype=None):
        import torch
        self.fn = fn
        self.n_grads = n_grads
        self.device = device
        self.group = group
        self.world_size = world_size
        self.streams = streams if streams is not None else CudaStreams(device)
        _, outs = fn.signature(1)
        self.grads = GradBuffer([s for s, _ in outs[:n_grads]], device, dtype=grads_dtype)
        self.kept = [torch.empty(s, dtype=grads_dtype or torch.float32, device=device) for s, _ in outs[n_grads:]]
        self.outputs = self.grads.views + self.kept
        self.buckets = layer_buckets(n_grads, per_bucket)
        # gradients become ready in reverse layer order: issue the last bucket first
        self.order = list(reversed(range(len(self.buckets))))
        self.events = [self.streams.new_event() for _ in range(n_grads)]
        self.comm = self.streams.new_stream() if world_size > 1 else None

    def step(self, inputs, seed, stream=None):
        st = stream or self.streams.current()
        self.fn.grad_run(inputs, seed=seed, outputs=self.outputs, stream=self.streams.handle(st),
                         events=self.events if self.comm is not None else None)
        if self.comm is None:
            return self.outputs
        works = allreduce_buckets(self.grads, self.buckets, self.group, self.order, self.comm, self.events,
                                  self.streams)
        for w in works:
            w.wait()  # makes the current stream wait for the collective
        self.streams.wait_stream(st, self.comm)
        return self.outputs


def assign_owners(sizes: Sequence[int], world: int) -> List[int]:
    """Owner rank of each gradient: largest first onto the least-loaded rank
    (deterministic, identical on every rank)."""
    load = [0] * world
    owner = [0] * len(sizes)
    for g in sorted(range(len(sizes)), key=lambda i: (-sizes[i], i)):
        r = min(range(world), key=lambda k: (load[k], k))
        owner[g] = r
        load[r] += sizes[g]
    return owner


class FusedReduceStep:
    """Data-parallel step with the gradient reduction fused into the kernels
    that produce the gradients (over NVLink peer
    memory): the flat gradient buffer is symmetric memory (one copy per rank,
    every rank can address every copy); each gradient has an owner rank
    (assign_owners), and every rank's dlvm_grad_run binds each gradient
    output as DLVM_F32_ADD into the OWNER's copy, so the dW GEMM epilogues /
    element-wise finalisers add their partial gradients straight into the
    owner's memory (red.global.add over NVLink) -- no separate all-reduce
    pass.  Protocol per step: zero this rank's copy, barrier (nobody adds
    before every copy is zeroed), grad_run, barrier (every contribution has
    landed); owners then hold the global-batch gradients of their tensors
    (seed 1/B_global, F15).  With `gather=True` each owner also copies its
    gradients into every peer's copy (so every rank ends with all of them,
    as after an all-reduce).  At world size 1 the owner is this rank and the
    step is a plain run accumulating into zeroed memory."""

    def __init__(self, fn, n_grads: int, device, group=None, gather: bool = True):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        from .dlvm import AddInto
        self.AddInto = AddInto
        self.fn, self.n_grads, self.device, self.gather = fn, n_grads, device, gather
        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        _, outs = fn.signature(1)
        self.shapes = [tuple(s) for s, _ in outs[:n_grads]]
        self.offsets, total = flat_layout(self.shapes)
        self.flat = symm.empty(max(total, 1), dtype=torch.float32, device=device)
        self.handle = symm.rendezvous(self.flat, self.group.group_name)
        self.ptrs = list(self.handle.buffer_ptrs)
        sizes = []
        for s in self.shapes:
            k = 1
            for d in s:
                k *= d
            sizes.append(k)
        self.sizes = sizes
        self.owner = assign_owners(sizes, self.world)
        self.views = [self.flat[o:o + k].view(s) for o, k, s in zip(self.offsets, sizes, self.shapes)]
        self.kept = [torch.empty(s, dtype=torch.float32, device=device) for s, _ in outs[n_grads:]]
        self.bindings = [AddInto(self.ptrs[self.owner[g]] + 4 * self.offsets[g], self.shapes[g])
                         for g in range(n_grads)] + self.kept

    def _barrier(self):
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return
        if hasattr(self.handle, "barrier"):
            self.handle.barrier()  # device-side barrier over the symmetric signal pads
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)

    def step(self, inputs, seed, stream=None):
        import torch
        st = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            self.flat.zero_()
            self._barrier()
            self.fn.grad_run(inputs, seed=seed, outputs=self.bindings, stream=st.cuda_stream)
            self._barrier()
            if self.gather and self.world > 1:
                for g in range(self.n_grads):
                    if self.owner[g] != self.rank:
                        continue
                    for r in range(self.world):
                        if r != self.rank:
                            peer = self.handle.get_buffer(r, self.shapes[g], torch.float32,
                                                          storage_offset=self.offsets[g])
                            peer.copy_(self.views[g])
                self._barrier()
        return self.views + self.kept


class ShardedSGD:
    """The update after a FusedReduceStep, sharded by gradient ownership
    ("reduce-scatter + a 1/N-sharded SGD update +
    all-gather of the bf16 weights").  The grad_run operands of every
    parameter -- bf16 copies of dot operands, f32 otherwise -- live in
    symmetric memory so owners can write every rank's copy.  The owner of a
    parameter keeps its fp32 master (the other ranks keep none: 1/N of the
    optimiser state per rank), updates it from the global gradient in its own
    copy of the fused gradient buffer with the SGD IR function
    (workloads-style `p - lr g`, one element-wise launch through the C ABI,
    writing the master and the operand copy), then copies the operand into
    every peer's copy (peer stores over NVLink: the all-gather); a barrier
    closes the step.  At world size 1 this is the plain full update."""

    def __init__(self, fused: "FusedReduceStep", host_params, is_dot_operand, lr: float, sgd_ir_fn):
        import numpy as np
        import torch
        import torch.distributed._symmetric_memory as symm
        from .dlvm import Function
        self.fused, self.lr = fused, lr
        dev = fused.device
        shapes = fused.shapes
        self.bf = [bool(b) for b in is_dot_operand]
        # one symmetric buffer per operand dtype, parameters at 256-byte aligned offsets
        self.handles, self.operands, self.offsets = {}, [None] * len(shapes), [0] * len(shapes)
        for dt, want in ((torch.bfloat16, True), (torch.float32, False)):
            idx = [i for i in range(len(shapes)) if self.bf[i] == want]
            if not idx:
                continue
            offs, total = flat_layout([shapes[i] for i in idx], align=128)
            buf = symm.empty(max(total, 1), dtype=dt, device=dev)
            h = symm.rendezvous(buf, fused.group.group_name)
            self.handles[want] = (buf, h)
            for i, o in zip(idx, offs):
                k = int(np.prod(shapes[i]))
                self.offsets[i] = o
                self.operands[i] = buf[o:o + k].view(shapes[i])
        for i, x in enumerate(host_params):
            self.operands[i].copy_(torch.from_numpy(np.ascontiguousarray(x)).to(dev).to(self.operands[i].dtype))
        self.owned = [i for i in range(len(shapes)) if fused.owner[i] == fused.rank]
        # fp32 masters of the owned parameters (f32 operands are their own masters)
        self.masters = {}
        for i in self.owned:
            self.masters[i] = (torch.from_numpy(np.ascontiguousarray(host_params[i])).to(dev) if self.bf[i]
                               else self.operands[i])
        self.sgd = None
        if self.owned:
            text = sgd_ir_fn([shapes[i] for i in self.owned], lr, [self.bf[i] for i in self.owned])
            self.sgd = Function(text, "sgd", None)
            self.sgd_in, self.sgd_out = [], []
            for i in self.owned:
                self.sgd_in += [self.masters[i], fused.views[i]]
                self.sgd_out.append(self.masters[i])
                if self.bf[i]:
                    self.sgd_out.append(self.operands[i])
            self.ws = self.sgd._workspace(0, dev)

    def step(self, stream=None):
        import torch
        f = self.fused
        st = stream or torch.cuda.current_stream(f.device)
        with torch.cuda.stream(st):
            if self.sgd is not None:
                self.sgd.run(self.sgd_in, outputs=self.sgd_out, workspace=self.ws, stream=st.cuda_stream)
            if f.world > 1:
                for i in self.owned:  # all-gather: the updated operand into every peer's copy
                    buf, h = self.handles[self.bf[i]]
                    for r in range(f.world):
                        if r != f.rank:
                            h.get_buffer(r, self.operands[i].shape, buf.dtype,
                                         storage_offset=self.offsets[i]).copy_(self.operands[i])
                f._barrier()
