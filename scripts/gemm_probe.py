"""Throughput of the CONV tcgen05 GEMM kernel (k_gemm_bf16 via the
cdn_debug_gemm_bf16 hook) on plain shapes: is the kernel itself far from the
tensor peak, or only the conv shapes?  Usage: python scripts/gemm_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1711_00244_b200 as cdn
    dev = torch.device("cuda:0")
    s = torch.cuda.Stream(dev)
    torch.cuda.set_stream(s)
    for M, N, K in ((8192 * 4, 256, 4096), (8192 * 4, 128, 4096), (46656, 128, 1600), (10816, 384, 2304),
                    (10816, 192, 1728), (193600, 96, 576), (148 * 128 * 4, 256, 8192)):
        A = torch.randint(-100, 100, (M, K), dtype=torch.int16, device=dev)
        Wt = torch.randint(-100, 100, (N, K), dtype=torch.int16, device=dev)
        bias = torch.zeros(N, dtype=torch.float32, device=dev)
        out = torch.empty((M, N), dtype=torch.float32, device=dev)
        for _ in range(3):
            cdn.debug_gemm_bf16(A, M, Wt, N, K, bias, False, out, N, stream=s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(s)
        for _ in range(reps):
            cdn.debug_gemm_bf16(A, M, Wt, N, K, bias, False, out, N, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = 2.0 * M * N * K / (ms / 1e3) / 1e12
        print(f"M={M} N={N} K={K}: {ms * 1e3:.1f} us, {tf:.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
