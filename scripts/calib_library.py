"""Calibration only (not part of the product or the bench): device time of
a library Blackwell attention kernel (flashinfer's CUTLASS sm100 FMHA,
JIT-built on the box) on the same shapes as scripts/probe_attn.py, so the
kernel's TFLOP/s can be read against what a library reaches on the same
power-capped B200.

    python scripts/calib_library.py
"""
import time

import torch


def bench(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    import flashinfer
    cases = [("causal S=32768 H=32 D=128", 32768, 32768, 32, 128, True),
             ("full 8192x16384 H=32 D=128", 8192, 16384, 32, 128, False)]
    for name, tq, tk, h, d, causal in cases:
        q = torch.randn(tq, h, d, device="cuda", dtype=torch.bfloat16)
        k = torch.randn(tk, h, d, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(tk, h, d, device="cuda", dtype=torch.bfloat16)
        qo = torch.tensor([0, tq], device="cuda", dtype=torch.int32)
        kv = torch.tensor([0, tk], device="cuda", dtype=torch.int32)
        t0 = time.time()
        fn = lambda: flashinfer.prefill.fmha_varlen(q, k, v, qo, kv, causal=causal, max_qo_len=tq)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        print(f"# first call (JIT) {time.time() - t0:.1f}s", flush=True)
        ms = bench(fn)
        flops = 4.0 * tq * tk * h * d * (0.5 if causal else 1.0)
        print(f"flashinfer-cutlass {name:30s} {ms:8.3f} ms {flops / ms / 1e9:9.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
