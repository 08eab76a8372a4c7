"""Validate the streamed backward's list kernels (decision -> vocab-major stream -> dE windows)
against a numpy model, reading them out of the workspace (CCE_STREAM_LISTS_ONLY=1)."""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2411_09009_b200 import _lib, ops  # noqa: E402

os.environ["CCE_STREAM_LISTS_ONLY"] = "1"
n, d, v = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(0)
e = torch.randn(n, d, device="cuda", generator=g).bfloat16()
c = (torch.randn(v, d, device="cuda", generator=g) / math.sqrt(d)).bfloat16()
t = torch.randint(0, v, (n,), device="cuda", generator=g)
lse_l, corr, st = ops.forward_tiles(e, c, t, -100, 0, 0.0, store_labels=False)
lse, _ = ops.merge_shards(lse_l[None], corr[None], t, -100)
up = ops.upstream(torch.ones((), device="cuda"), t, -100, "mean")
inv = torch.empty_like(st.perm)
inv[st.perm.long()] = torch.arange(st.perm.shape[0], dtype=torch.int32, device="cuda")
lib = _lib.load()
slots = ops.stream_ring_slots()
ws_bytes = lib.cce_bwd_stream_workspace_bytes(n, d, v, slots)
ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
ring = torch.empty(slots * ops.SHAT_TILE_BYTES, dtype=torch.uint8, device="cuda")
de = torch.zeros(n, d, dtype=torch.bfloat16, device="cuda")
cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
P = ops._p
_lib.check(lib.cce_bwd_stream(P(e), 1, P(c), P(torch.empty_like(c)), P(st.perm_padded), P(inv), P(st.row_map),
                              P(st.n_valid), P(st.pos), P(lse), P(up), P(st.tile_max), n, d, v, 0.0, 2.0 ** -12, 0,
                              P(ring), slots, P(ws), ws_bytes, P(de), 0, P(None), P(cnt), P(None),
                              ops._stream(e.device)), "cce_bwd_stream")
torch.cuda.synchronize()
offs = (ctypes.c_int64 * 13)()
W = lib.cce_bwd_stream_debug_layout(n, d, v, slots, offs)
offs = list(offs)
buf = ws.cpu().numpy()
nt, mt = -(-n // 128), -(-v // 256)


def arr(k, count, dtype, width=1):
    a = np.frombuffer(buf[offs[k]:offs[k] + count * width * np.dtype(dtype).itemsize].tobytes(), dtype=dtype)
    return a.reshape(count, width) if width > 1 else a


keep = arr(0, nt * mt, np.uint8).reshape(mt, nt)
ctrl = arr(7, 16, np.int32)
K = int(ctrl[0])
print("kept", K, "keep.sum", int(keep.sum()), "dC segs", ctrl[1], "pairs", ctrl[2], "dE segs", ctrl[3], "W", W)
items = arr(1, K, np.int32, 2)
ref_items = np.array([(nn, m) for m in range(mt) for nn in range(nt) if keep[m, nn]], dtype=np.int32).reshape(-1, 2)
print("items ok", np.array_equal(items, ref_items))
nw = -(-K // W)
wcnt = arr(2, nw * nt, np.int32).reshape(nw, nt)
ref_wcnt = np.zeros((nw, nt), np.int32)
for i in range(K):
    ref_wcnt[i // W, items[i, 0]] += 1
print("wcnt ok", np.array_equal(wcnt, ref_wcnt))
sidx = arr(4, K, np.int32)
ref_sidx = np.concatenate([[i for i in range(w * W, min(K, (w + 1) * W)) if items[i, 0] == nn]
                           for w in range(nw) for nn in range(nt)]).astype(np.int32)
print("sidx ok", np.array_equal(sidx, ref_sidx), "first diffs", np.nonzero(sidx != ref_sidx)[0][:5])
S = int(ctrl[3])
eseg = arr(5, S, np.int32, 4)
eaux = arr(6, S, np.int32, 2)
ref = []
nsp = [(ref_wcnt[:, nn] > 0).sum() for nn in range(nt)]
start = 0
k_of = {}
for w in range(nw):
    a = w * W
    for nn in range(nt):
        cc = ref_wcnt[w, nn]
        if cc:
            k_of[nn] = k_of.get(nn, -1) + 1
            ref.append((nn, a, cc, k_of[nn], nsp[nn], nn))
        a += cc
ref = np.array(ref, np.int32)
print("eseg ok", np.array_equal(eseg, ref[:, :4]), "eaux ok", np.array_equal(eaux, ref[:, 4:]), S, len(ref))
