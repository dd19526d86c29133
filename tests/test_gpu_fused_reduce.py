"""Gradient outputs accumulated in place (DLVM_F32_ADD, dlvm.h): the fused
gradient reduction of the data-parallel path.  On
one GPU: accumulation into pre-filled memory equals prefill + the stored
result (GEMM epilogue, split-K sum step and finalize paths), outputs read
back by a later launch are refused, and FusedReduceStep at world size 1
equals the plain run.  On >= 2 GPUs (skipped otherwise): every rank adds its
shard gradients into the owners' peer memory and the result equals the
oracle's global-batch gradient (F15)."""

import os
import socket

import numpy as np
import pytest

import oracle
import workloads as W
from helpers import assert_normwise

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("batch,prec", [(96, "f32"), (256, "bf16"), (8192, "bf16")])
def test_accumulated_outputs_equal_prefill_plus_result(batch, prec):
    import torch
    import paper_1711_03016_b200 as P
    w = W.c3(batch, layers=[(512, 512, "relu"), (512, 256, None)])
    f = P.Function(w.text, w.fn, w.grad, dot_precision=prec)
    if batch == 8192:
        assert "K split" in f.print(3)  # the split-K sum step stores the dW
    dev = torch.device("cuda:0")
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    ref = f.grad_run(ins, seed=seed)
    gen = torch.Generator(device=dev).manual_seed(7)
    pre = [torch.randn(r.shape, device=dev, generator=gen) for r in ref[:-1]]
    acc = [p.clone() for p in pre]
    outs = [P.AddInto(a) for a in acc] + [torch.empty_like(ref[-1])]
    f.grad_run(ins, seed=seed, outputs=outs)
    torch.cuda.synchronize()
    for k, (a, p, r) in enumerate(zip(acc, pre, ref)):
        want = p + r  # one fp32 rounding, as the hardware red.add
        assert torch.equal(a, want), (k, float((a - want).abs().max()))
    assert torch.equal(outs[-1], ref[-1])


def test_accumulated_output_read_by_a_later_launch_is_refused():
    import torch
    import paper_1711_03016_b200 as P
    X, Wt, Y = "<128 x 64 x f32>", "<64 x 32 x f32>", "<128 x 32 x f32>"
    text = (f'module "r"\nstage raw\nfunc @f: ({X}, {Wt}) -> ({X}, {Y}) {{\n'
            f"'entry(%x: {X}, %w: {Wt}):\n    %h = tanh %x: {X}\n    %y = dot %h: {X}, %w: {Wt}\n"
            f"    return (%h: {X}, %y: {Y})\n}}\n")
    f = P.Function(text, "f", None)
    dev = torch.device("cuda:0")
    x, wt = torch.randn(128, 64, device=dev), torch.randn(64, 32, device=dev)
    h, y = torch.zeros(128, 64, device=dev), torch.zeros(128, 32, device=dev)
    with pytest.raises(P.DlvmError) as e:
        f.run([x, wt], outputs=[P.AddInto(h), y])
    assert e.value.status == 3
    f.run([x, wt], outputs=[h, P.AddInto(y)])  # the dot's result is terminal: fine
    torch.cuda.synchronize()
    torch.testing.assert_close(y, torch.tanh(x) @ wt, rtol=1e-5, atol=1e-5)


def test_fused_reduce_step_world_size_one():
    import torch
    import torch.distributed as dist
    import paper_1711_03016_b200 as P
    from paper_1711_03016_b200.dp import DataParallelStep, FusedReduceStep
    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    w = W.c3(256, layers=[(512, 512, "relu"), (512, 256, None)])
    f = P.Function(w.text, w.fn, w.grad, dot_precision="bf16")
    dev = torch.device("cuda:0")
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs()]
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    n = 2 * len(w.layers)
    plain = [o.clone() for o in DataParallelStep(f, n, dev).step(ins, seed)]
    fused = FusedReduceStep(f, n, dev)
    for _ in range(2):  # the buffer is re-zeroed every step
        got = fused.step(ins, seed)
    torch.cuda.synchronize()
    for a, b in zip(got, plain):
        assert torch.equal(a, b)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import paper_1711_03016_b200 as P
    from paper_1711_03016_b200.dp import FusedReduceStep
    GB = 256
    w = W.c3(GB // world, global_batch=GB, layers=[(256, 512, "relu"), (512, 128, None)])
    f = P.Function(w.text, w.fn, w.grad, dot_precision="bf16")
    ins = [torch.from_numpy(x).to(dev) for x in w.inputs(row_offset=rank * w.batch)]
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    step = FusedReduceStep(f, 2 * len(w.layers), dev)
    outs = step.step(ins, seed)
    torch.cuda.synchronize(dev)
    grads = [o.double().cpu().numpy() for o in outs[:-1]]
    # sharded update + all-gather: every rank ends with the same operands
    from paper_1711_03016_b200.dp import ShardedSGD
    host = w.inputs(row_offset=rank * w.batch)
    dot_op = [a.name.startswith("w") for a in w.args[1:-1]]
    step2 = FusedReduceStep(f, 2 * len(w.layers), dev, gather=False)
    upd = ShardedSGD(step2, host[1:-1], dot_op, 1e-3, W.sgd_ir)
    step2.step([ins[0]] + upd.operands + [ins[-1]], seed)
    upd.step()
    torch.cuda.synchronize(dev)
    ops = [o.float().cpu() for o in upd.operands]
    gathered = [None] * world
    dist.all_gather_object(gathered, [o.numpy() for o in ops])
    if rank == 0:
        for other in gathered[1:]:
            for a, b in zip(gathered[0], other):
                assert np.array_equal(a, b)
        out.put(grads)
    dist.destroy_process_group()


def test_fused_reduce_two_ranks_equals_global_gradient():
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = W.c3(256, layers=[(256, 512, "relu"), (512, 128, None)])
    m = oracle.parse(w.text)
    ref = oracle.run(m, w.grad, [x.astype(np.float64) for x in w.inputs()] + [np.float64(w.seed())],
                     dot_policy="bf16")
    for k, (g, r) in enumerate(zip(got, ref[:-1])):
        assert_normwise(g, r, what=f"fused dp grad out{k}")


def test_sharded_sgd_training_world_size_one_equals_plain_step():
    """Two training steps (fwd+adjoint, gradient reduction, SGD) of a small
    tanh MLP: FusedReduceStep + ShardedSGD (owners update their fp32 masters
    and broadcast the operand copies; at world size 1 rank 0 owns all) give
    bit-identical weights, operand copies and losses to DataParallelStep + the
    full SGD IR function."""
    import torch
    import torch.distributed as dist
    import paper_1711_03016_b200 as P
    from paper_1711_03016_b200.dp import DataParallelStep, FusedReduceStep, ShardedSGD
    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    w = W._mlp_workload(5, "c5s", 256, [(512, 512, "tanh")] * 2, ("normal",), ("uniform", -0.5, 0.5),
                        1.0 / 256, "bf16", 256)
    dev = torch.device("cuda:0")
    host = w.inputs()
    n = 2 * len(w.layers)
    dot_op = [a.name.startswith("w") for a in w.args[1:-1]]
    f = P.Function(w.text, w.fn, w.grad, dot_precision="bf16")
    seed = torch.tensor(np.float32(w.seed()), device=dev)
    x = torch.from_numpy(host[0]).to(dev).to(torch.bfloat16)
    t = torch.from_numpy(host[-1]).to(dev)
    # plain: all-reduce path (world 1) + the full SGD IR function
    shapes = [a.shape for a in w.args[1:-1]]
    sgd = P.Function(W.sgd_ir(shapes, 1e-3, dot_op), "sgd", None)
    masters = [torch.from_numpy(hp).to(dev) for hp in host[1:-1]]
    ops = [m.to(torch.bfloat16) if b else m for m, b in zip(masters, dot_op)]
    dps = DataParallelStep(f, n, dev)
    sgd_in, sgd_out = [], []
    for j in range(n):
        sgd_in += [masters[j], dps.grads.views[j]]
        sgd_out.append(masters[j])
        if dot_op[j]:
            sgd_out.append(ops[j])
    losses_a = []
    for _ in range(2):
        outs = dps.step([x] + ops + [t], seed)
        losses_a.append(outs[-1].clone())
        sgd.run(sgd_in, outputs=sgd_out)
    # fused reduction + sharded update
    fused = FusedReduceStep(f, n, dev, gather=False)
    upd = ShardedSGD(fused, host[1:-1], dot_op, 1e-3, W.sgd_ir)
    losses_b = []
    for _ in range(2):
        outs = fused.step([x] + upd.operands + [t], seed)
        losses_b.append(outs[-1].clone())
        upd.step()
    torch.cuda.synchronize()
    for a, b in zip(losses_a, losses_b):
        assert torch.equal(a, b)
    for j in range(n):
        assert torch.equal(ops[j], upd.operands[j]), j
        assert torch.equal(masters[j], upd.masters[j]), j
