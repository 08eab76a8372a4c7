"""Where the default training step leaves the GPU idle: torch.profiler (CUPTI) trace of a few
steps, then the gaps between consecutive kernels (any stream) longer than GAP_US, with the
kernels on either side.  Usage: python scripts/gap_probe.py [config]"""
import json
import math
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2411_09009_b200 import linear_cross_entropy  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gemma2-2b"
gap_us = float(os.environ.get("GAP_US", 8))
n, d, v, cap, pad, sigma = bench.CONFIGS[cfg]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
e = torch.randn(n, d, device=dev, generator=g).bfloat16().requires_grad_(True)
c = (torch.randn(v, d, device=dev, generator=g) * sigma / math.sqrt(d)).bfloat16().requires_grad_(True)
t = torch.randint(0, v, (n,), device=dev, generator=g)


def step():
    e.grad = c.grad = None
    linear_cross_entropy(e, c, t, softcap=cap or None).backward()


for _ in range(4):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
path = "/tmp/gap_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
kern = sorted([x for x in ev if x.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in x],
              key=lambda x: x["ts"])
span = kern[-1]["ts"] + kern[-1]["dur"] - kern[0]["ts"]
busy_end = kern[0]["ts"]
gaps = []
for k in kern:
    if k["ts"] > busy_end + gap_us:
        gaps.append((k["ts"] - busy_end, prev["name"][:60], k["name"][:60]))
    if k["ts"] + k["dur"] > busy_end:
        busy_end = k["ts"] + k["dur"]
        prev = k
total_gap = sum(x[0] for x in gaps)
print(f"{cfg}: 3 steps span {span / 1e3:.2f} ms, {len(kern)} kernels/copies, idle gaps > {gap_us} us: "
      f"{len(gaps)} totalling {total_gap / 1e3:.3f} ms")
for gp, a, b in sorted(gaps, reverse=True)[:25]:
    print(f"  {gp:8.1f} us  after {a}  before {b}")
