"""Forward variants of the training path at one head, timed on one box (CUDA events):
tiles (sorted classifier copy), gather (cp.async row gathers in the logit-tile kernel), stream
(vocabulary groups of CCE_FWD_GROUP_MB gathered per launch)."""
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2411_09009_b200 import ops  # noqa: E402

CFG = {"gemma2-2b": (8192, 2304, 256000, 0.0), "gemma2-9b": (32768, 3584, 256000, 30.0),
       "llama3-8b": (16384, 4096, 128256, 0.0), "gpt2": (4096, 768, 50257, 0.0)}
name = sys.argv[1] if len(sys.argv) > 1 else "gemma2-2b"
n, d, v, cap = CFG[name]
g = torch.Generator(device="cuda").manual_seed(0)
e = torch.randn(n, d, device="cuda", generator=g).bfloat16()
c = (torch.randn(v, d, device="cuda", generator=g) / math.sqrt(d)).bfloat16()
t = torch.randint(0, v, (n,), device="cuda", generator=g)
reps = int(os.environ.get("REPS", "5"))
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tiles", "gather", "stream:24", "stream:48", "stream:96"]
for var in variants:
    kind, _, mb = var.partition(":")
    if mb:
        os.environ["CCE_FWD_GROUP_MB"] = mb
    fn = {"tiles": lambda: ops.forward_tiles(e, c, t, -100, 0, cap, store_labels=False),
          "gather": lambda: ops.forward_gather(e, c, t, -100, 0, cap),
          "stream": lambda: ops.forward_stream(e, c, t, -100, 0, cap)}[kind]
    out = fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name} {var}: {a.elapsed_time(b) / reps:.3f} ms", flush=True)
