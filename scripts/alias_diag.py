"""Diagnostics for test_dc_aliasing_sorted_copy_is_bit_identical[1-1]: which outputs differ between
a separate dC buffer and dC over the sorted copy on the overflow fallback, and whether each is
deterministic."""
import math, os, sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from oracle import cce_oracle as O
import test_gpu_parity as T
from paper_2411_09009_b200 import ops

rng = np.random.default_rng(31)
n, d, v = 3000, 64, 20000
e = O.round_to_bf16(rng.standard_normal((n, d)).astype(np.float32))
c = O.round_to_bf16((rng.standard_normal((v, d)) * 3.0 / math.sqrt(d)).astype(np.float32))
x = rng.integers(0, v, n)
x[::11] = -1
os.environ["CCE_STORE_LABELS"] = os.environ.get("STORE", "1")
os.environ["CCE_SHAT_BUDGET_MB"] = "1"
res = {}
for alias in ("0", "1", "0", "1"):
    os.environ["CCE_ALIAS_DC"] = alias
    r = T._run(e, c, x, path="tiles")
    res.setdefault(alias, []).append(r)
names = ["loss", "de", "dc", "cnt", "perm"]
for a in ("0", "1"):
    print("alias", a, "deterministic:", [np.array_equal(p, q) for p, q in zip(res[a][0][:5], res[a][1][:5])])
for i, (p, q) in enumerate(zip(res["0"][0][:5], res["1"][0][:5])):
    if not np.array_equal(p, q):
        diff = p != q
        print(names[i], "differs at", int(diff.sum()), "of", p.size, "rows", np.unique(np.nonzero(diff)[0])[:20],
              "max abs", float(np.abs(p.astype(np.float64) - q).max()), "max", float(np.abs(p).max()))
