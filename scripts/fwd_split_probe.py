"""The bounded forward's cost of cutting the sweep into vocabulary-group launches: the same logit
tiles over one sorted classifier copy, swept by one launch (the whole vocabulary) or by one launch
per group (ops.fwd_group_tiles), no gathers in either; CUDA events, alternating rounds.
Usage: python scripts/fwd_split_probe.py [config]"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2411_09009_b200 import _lib, ops  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gemma2-2b"
reps = int(os.environ.get("REPS", 4))
n, d, v, cap, pad, sigma = bench.CONFIGS[cfg]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
e = torch.randn(n, d, device=dev, generator=g).bfloat16()
c = (torch.randn(v, d, device=dev, generator=g) * sigma / math.sqrt(d)).bfloat16()
t = torch.randint(0, v, (n,), device=dev, generator=g)
lib = _lib.load()
row_map, n_valid, perm, perm_padded, pos, _, _ = ops.prepare_order(e, c, t, -100, 0, True, None, with_inverse=True)
c_t = ops.gather_rows(c, perm, v)
mt = -(-v // 256)
tile_max = torch.empty(-(-n // 128) * mt * 128, dtype=torch.float32, device=dev)
correct = torch.zeros(n, dtype=torch.float32, device=dev)
stream = ops._stream(dev)


def sweep(groups):
    splits = [lib.cce_fwd_splits(n, d, v1 - v0) for v0, v1 in groups]
    parts = torch.empty(1 + sum(splits), n, 2, dtype=torch.float32, device=dev)
    off = 1
    for (v0, v1), sp in zip(groups, splits):
        ws = parts[off:off + sp]
        _lib.check(lib.cce_fwd_group_ex(ops._p(e), 1, ops._p(c_t[v0:v1]), ops._p(row_map), ops._p(n_valid),
                                        ops._p(pos), v0, n, d, v1 - v0, v, float(cap or 0.0), ops._p(ws),
                                        sp * n * 8, ops._p(None), ops._p(correct), ops._p(tile_max), 3, stream),
                   "cce_fwd_group_ex")
        off += sp


def timed(groups):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        sweep(groups)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


gt = ops.fwd_group_tiles(d, mt, n, ops._sm_count(dev))
variants = {"one launch": [(0, v)]}
for tiles in sorted({gt, 2 * gt, 4 * gt, ops.fwd_group_tiles(d, mt)}):
    variants[f"groups of {tiles}"] = [(m0 * 256, min(v, (m0 + tiles) * 256)) for m0 in range(0, mt, tiles)]
for grp in variants.values():
    sweep(grp)
flops = 2.0 * n * v * d
res = {k: [] for k in variants}
for r in range(int(os.environ.get("ROUNDS", 8))):  # interleaved: clocks drift under the power cap
    for k, gv in variants.items():
        res[k].append(timed(gv))
for k, xs in res.items():
    xs = sorted(xs)
    print(f"{cfg} {k:>16}: median {xs[len(xs) // 2]:.3f} ms  min {xs[0]:.3f} ms  "
          f"({flops / (xs[len(xs) // 2] / 1e3) / 1e12:.0f} TF/s at the median)")
