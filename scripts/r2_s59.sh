#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for e in "X=1" "CCE_FWD_OVERLAP=0" "X=1"; do echo "$e: $(env $e timeout 300 python scripts/host_overhead.py gpt2 2>&1 | tail -2 | tr '\n' ' ')"; done
echo "gemma: $(timeout 300 python scripts/host_overhead.py gemma2-2b 2>&1 | tail -2 | tr '\n' ' ')"
timeout 300 python - <<'PY'
import cProfile, pstats, math, torch, sys
sys.path.insert(0, ".")
import bench
from paper_2411_09009_b200 import linear_cross_entropy
n, d, v, cap, pad, sigma = bench.CONFIGS["gpt2"]
e = torch.randn(n, d, device="cuda").bfloat16().requires_grad_(True)
c = (torch.randn(v, d, device="cuda") / math.sqrt(d)).bfloat16().requires_grad_(True)
t = torch.randint(0, v, (n,), device="cuda")
def step():
    e.grad = c.grad = None
    linear_cross_entropy(e, c, t).backward()
for _ in range(10): step()
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(20): step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
PY
