"""Forward over the backward's tile order: sorted/compacted copies (forward_tiles) vs cp.async
row gathers (forward_gather).  Checks bit-identity and times both (CUDA events)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2411_09009_b200 import ops  # noqa: E402

CFG = {"gemma2-2b": (8192, 2304, 256000, 0.0, 0.0), "llama3-8b": (16384, 4096, 128256, 0.0, 0.25),
       "gemma2-9b": (32768, 3584, 256000, 30.0, 0.0), "nemo-12b": (65536, 5120, 131072, 0.0, 0.0),
       "gpt2": (4096, 768, 50257, 0.0, 0.0)}


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


for name in sys.argv[1:] or ["gpt2", "gemma2-2b", "llama3-8b", "gemma2-9b", "nemo-12b"]:
    n, d, v, cap, pad = CFG[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    e = torch.randn(n, d, device="cuda", generator=g).bfloat16()
    c = (torch.randn(v, d, device="cuda", generator=g) / math.sqrt(d)).bfloat16()
    t = torch.randint(0, v, (n,), device="cuda", generator=g)
    if pad:
        t[(torch.arange(n, device="cuda") % 4096) >= int(4096 * (1 - pad))] = -100
    reps = 5 if n * v * d > 2e13 else 10
    ops.KERNEL_EVENTS = {}
    ms_t, (l1, c1, s1) = timed(lambda: ops.forward_tiles(e, c, t, -100, 0, cap, store_labels=False), reps)
    k_t = sum(a.elapsed_time(b) for a, b in ops.KERNEL_EVENTS["fwd"][1:]) / reps
    ops.KERNEL_EVENTS = {}
    ms_g, (l2, c2, s2) = timed(lambda: ops.forward_gather(e, c, t, -100, 0, cap), reps)
    k_g = sum(a.elapsed_time(b) for a, b in ops.KERNEL_EVENTS["fwd"][1:]) / reps
    ops.KERNEL_EVENTS = None
    valid = t != -100
    same = (torch.equal(l1[valid], l2[valid]) and torch.equal(c1[valid], c2[valid])
            and torch.equal(s1.tile_max, s2.tile_max))
    fl = 2.0 * int(valid.sum()) * v * d
    print(f"{name}: copies {ms_t:.3f} ms (kernel {k_t:.3f} ms, {fl / k_t / 1e9:.0f} TF/s) | gather {ms_g:.3f} ms "
          f"(kernel {k_g:.3f} ms, {fl / k_g / 1e9:.0f} TF/s) | bit-identical {same}", flush=True)
    del e, c, t, l1, l2, c1, c2, s1, s2
    torch.cuda.empty_cache()
