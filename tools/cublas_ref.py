#!/usr/bin/env python
"""cuBLAS (torch.matmul, bf16 in / fp32 accumulate / bf16 out) on the c4
GEMM shapes, for comparison with the tcgen05 kernels' mainloops: ms and
TFLOP/s per shape (CUDA events, 20 runs after warm-up).  Library GEMMs
here are a yardstick only; the product path never calls them.
usage: cublas_ref.py"""
import torch

SHAPES = [("z1 65536x4096x4096", 65536, 4096, 4096), ("z3 65536x1000x4096", 65536, 1000, 4096),
          ("d11 65536x4096x1000", 65536, 4096, 1000), ("d20 4096x4096x65536", 4096, 4096, 65536),
          ("sq 8192^3", 8192, 8192, 8192)]


def main():
    dev = torch.device("cuda:0")
    for name, M, N, K in SHAPES:
        a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
        b = torch.randn(K, N, device=dev, dtype=torch.bfloat16)
        for _ in range(5):
            c = a @ b
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            c = a @ b
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{name:24s} {ms:8.4f} ms  {2.0 * M * N * K / ms / 1e9:8.1f} TFLOP/s", flush=True)
        del a, b, c


if __name__ == "__main__":
    main()
