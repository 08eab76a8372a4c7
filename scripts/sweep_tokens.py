"""Throughput vs batch size at one head shape (default Gemma-2-2B: D=2304, V=256000): device time
of fwd+bwd per step (CUDA events over K steps after warm-up), tokens/s, the forward kernel's
TFLOP/s and the kept-tile fraction.  Usage: python scripts/sweep_tokens.py [D] [V] [N...]"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_09009_b200 import linear_cross_entropy, ops

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2304
v = int(sys.argv[2]) if len(sys.argv) > 2 else 256000
ns = [int(x) for x in sys.argv[3:]] or [2048, 4096, 8192, 16384, 32768]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
c = (torch.randn(v, d, device=dev, generator=g) / math.sqrt(d)).bfloat16().requires_grad_(True)
for n in ns:
    e = torch.randn(n, d, device=dev, generator=g).bfloat16().requires_grad_(True)
    t = torch.randint(0, v, (n,), device=dev, generator=g)

    def step():
        e.grad = c.grad = None
        linear_cross_entropy(e, c, t).backward()

    for _ in range(4):
        step()
    torch.cuda.synchronize()
    steps = max(5, int(2e5 // n))
    ops.KERNEL_EVENTS = {}
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    fwd = sum(x.elapsed_time(y) for x, y in ops.KERNEL_EVENTS["fwd"]) / steps
    ops.KERNEL_EVENTS = None
    k = ops.LAST_COUNTERS["counters"].tolist()
    tiles = -(-n // 128) * -(-v // 256)
    print(json.dumps({"N": n, "D": d, "V": v, "ms_per_step": round(ms, 3), "tokens_per_s": round(n / ms * 1e3),
                      "fwd_ms": round(fwd, 3), "fwd_tflops": round(2 * n * v * d / fwd / 1e9, 1),
                      "kept_frac": round(k[0] / tiles, 4)}), flush=True)
    del e, t
