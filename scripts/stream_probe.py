"""Time the streamed backward against the stored-S-hat backward on one head (CUDA events)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2411_09009_b200 import ops  # noqa: E402

CFG = {"gemma2-2b": (8192, 2304, 256000, 0.0), "llama3-8b": (16384, 4096, 128256, 0.0),
       "gemma2-9b": (32768, 3584, 256000, 30.0), "gpt2": (4096, 768, 50257, 0.0)}


def ev():
    return torch.cuda.Event(enable_timing=True)


for name in sys.argv[1:] or ["gemma2-2b"]:
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

    def stream():
        return ops.backward_stream(e, True, c, st.perm_padded, inv, st.row_map, st.n_valid, st.pos, st.tile_max,
                                   lse, up, softcap=cap)

    def stored():
        return ops.backward_tiles(st, t, lse, up, ignore_index=-100, reuse_state=True)

    for nm, fn in (("stored", stored), ("stream", stream)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        a, b = ev(), ev()
        a.record()
        reps = 5
        for _ in range(reps):
            out = fn()
        b.record()
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base
        k = out[2].tolist()
        print(f"{name} {nm}: {a.elapsed_time(b) / reps:.3f} ms, kept {k[0]}, peak over base {peak / 2**20:.0f} MiB",
              flush=True)
    de1, dc1, _ = stream()
    de2, dc2, _ = stored()
    torch.cuda.synchronize()
    r = lambda x, y: float((x.float() - y.float()).abs().max() / y.float().abs().max())
    print(f"{name} stream vs stored: dE {r(de1, de2):.2e} dC {r(dc1, dc2):.2e}", flush=True)
    del e, c, t, st
    torch.cuda.empty_cache()
