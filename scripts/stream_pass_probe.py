"""Streamed backward at one head: dE-only / dC-only / both, with and without the dC-over-sorted-copy
aliasing, checked against the stored-S-hat backward and timed (CUDA events)."""
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2411_09009_b200 import ops  # noqa: E402

CFG = {"gemma2-2b": (8192, 2304, 256000, 0.0), "gpt2": (4096, 768, 50257, 0.0), "small": (2048, 512, 40000, 0.0),
       "llama": (8192, 4096, 128256, 0.0), "d1536": (8192, 1536, 128000, 0.0),
       "gemma9b": (32768, 3584, 256000, 30.0), "gemma2b-cap": (8192, 2304, 256000, 30.0)}
name = sys.argv[1] if len(sys.argv) > 1 else "gemma2-2b"
n, d, v, cap = CFG[name]
g = torch.Generator(device="cuda").manual_seed(0)
e = torch.randn(n, d, device="cuda", generator=g).bfloat16()
c = (torch.randn(v, d, device="cuda", generator=g) / math.sqrt(d)).bfloat16()
t = torch.randint(0, v, (n,), device="cuda", generator=g)
lse_l, corr, st = ops.forward_tiles(e, c, t, -100, 0, cap, store_labels=False)
lse, _ = ops.merge_shards(lse_l[None], corr[None], t, -100)
up = ops.upstream(torch.ones((), device="cuda"), t, -100, "mean")
inv = torch.empty_like(st.perm)
inv[st.perm.long()] = torch.arange(st.perm.shape[0], dtype=torch.int32, device="cuda")
rde, rdc, rcnt = ops.backward_tiles(st, t, lse, up, ignore_index=-100, reuse_state=True)
torch.cuda.synchronize()
r = lambda x, y: float((x.float() - y.float()).abs().max() / y.float().abs().max())
reps = int(os.environ.get("REPS", "5"))
MODES = {"de": ("dE only", True, False), "dc": ("dC only", False, True), "both": ("both", True, True)}
seq = [m.split(":") for m in (sys.argv[2].split(",") if len(sys.argv) > 2 else
                              ["de:0", "dc:0", "both:0", "de:1", "dc:1", "both:1"])]
for mode, alias in seq:
    os.environ["CCE_STREAM_ALIAS"] = alias
    for nm, wde, wdc in (MODES[mode],):
        fn = lambda: ops.backward_stream(e, True, c, st.perm_padded, inv, st.row_map, st.n_valid, st.pos,
                                         st.tile_max, lse, up, softcap=cap, want_de=wde, want_dc=wdc)
        de, dc, cnt = fn()
        torch.cuda.synchronize()
        errs = (f"dE {r(de, rde):.2e} " if wde else "") + (f"dC {r(dc, rdc):.2e} " if wdc else "")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        print(f"{name} alias={alias} {nm}: {a.elapsed_time(b) / reps:.3f} ms  {errs} kept {cnt[0].item()} "
              f"(ref {rcnt[0].item()})", flush=True)
