"""Per-unit timeline of the dE consumers of the streamed backward (libcce_b200_prof.so)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
prof = torch.zeros(8 * 400000, dtype=torch.int64, device="cuda")
os.environ["CCE_STREAM_PROF_PTR"] = str(prof.data_ptr())
from paper_2411_09009_b200 import ops  # noqa: E402

n, d, v = 8192, 2304, 256000
g = torch.Generator(device="cuda").manual_seed(0)
e = torch.randn(n, d, device="cuda", generator=g).bfloat16()
c = (torch.randn(v, d, device="cuda", generator=g) / math.sqrt(d)).bfloat16()
t = torch.randint(0, v, (n,), device="cuda", generator=g)
lse_l, corr, st = ops.forward_tiles(e, c, t, -100, 0, 0.0, store_labels=False)
lse, _ = ops.merge_shards(lse_l[None], corr[None], t, -100)
up = ops.upstream(torch.ones((), device="cuda"), t, -100, "mean")
inv = torch.empty_like(st.perm)
inv[st.perm.long()] = torch.arange(st.perm.shape[0], dtype=torch.int32, device="cuda")
mode = sys.argv[1] if len(sys.argv) > 1 else "de"
for _ in range(3):
    prof.zero_()
    ops.backward_stream(e, True, c, st.perm_padded, inv, st.row_map, st.n_valid, st.pos, st.tile_max, lse, up,
                        want_de=True, want_dc=(mode == "both"))
    torch.cuda.synchronize()
P = prof.view(-1, 8).cpu().numpy()
used = P[:, 0] > 0
P = P[used]
t0 = P[:, 0].min()
T = (P[:, :6] - t0) / 1000.0  # us
T[P[:, :6] == 0] = np.nan
bid = P[:, 6]
start = (P[:, 7] & 0xffffffff)
W = int(os.environ.get("CCE_STREAM_WINDOW", 256))
win = start // W
print(f"units {len(P)}, ctas {len(np.unique(bid))}, windows {win.max() + 1}, span {np.nanmax(T):.0f} us")
cols = ["prod_start", "loads_done", "epi_begin", "acc_full", "chain_ok", "epi_end"]
for k in range(1, 6):
    dlt = T[:, k] - T[:, k - 1]
    print(f"{cols[k-1]}->{cols[k]}: mean {np.nanmean(dlt):.2f} us, p50 {np.nanpercentile(dlt, 50):.2f}, p90 {np.nanpercentile(dlt, 90):.2f}, max {np.nanmax(dlt):.1f}")
for w in [0, 1, 2, 10, 20, int(win.max())]:
    m = win == w
    print(f"window {w}: units {m.sum()}, loads from {np.nanmin(T[m,0]):.0f} to {np.nanmax(T[m,1]):.0f} us, "
          f"epilogues end {np.nanmin(T[m,5]):.0f}..{np.nanmax(T[m,5]):.0f} us")
# per CTA busy
b0 = bid == bid.min()
print("first CTA units (prod_start, loads_done, acc_full, chain_ok, epi_end):")
for r in T[b0][:12]:
    print("  " + " ".join(f"{x:8.1f}" for x in [r[0], r[1], r[3], r[4], r[5]]))
