"""Time torch SDPA (cuDNN / flash backends) dense causal attention on a BASELINE shape, so its kernel
can be captured by ncu beside ours (external sanity reference, not the product path).

usage: python tools/sdpa_probe.py [--n 32768] [--hq 32] [--hkv 8] [--d 128] [--reps 3]"""
import argparse

import torch
import torch.nn.functional as F

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--backend", default="cudnn", choices=["cudnn", "flash", "any"])
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(1, a.hq, a.n, a.d, device="cuda", dtype=torch.bfloat16, generator=g)
k = torch.randn(1, a.hkv, a.n, a.d, device="cuda", dtype=torch.bfloat16, generator=g)
v = torch.randn(1, a.hkv, a.n, a.d, device="cuda", dtype=torch.bfloat16, generator=g)
k = k.repeat_interleave(a.hq // a.hkv, dim=1)
v = v.repeat_interleave(a.hq // a.hkv, dim=1)
from torch.nn.attention import SDPBackend, sdpa_kernel

be = {"cudnn": [SDPBackend.CUDNN_ATTENTION], "flash": [SDPBackend.FLASH_ATTENTION],
      "any": [SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION]}[a.backend]
with sdpa_kernel(be):
    for _ in range(a.reps):
        F.scaled_dot_product_attention(q, k, v, is_causal=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        F.scaled_dot_product_attention(q, k, v, is_causal=True)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
fl = 4 * a.d * a.hq * a.n * (a.n + 1) / 2
print(f"sdpa[{a.backend}] N={a.n} Hq={a.hq} d={a.d}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s")
