"""Developer probe: run the CUDA path on small shapes and print errors vs the CPU oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2411_09009_b200 import ops
from oracle import cce_oracle as O

def case(n, d, v, seed=0, sigma=1.0, ignore_frac=0.0, softcap=0.0, sort=True, eps=O.EPSILON_DEFAULT):
    g = torch.Generator().manual_seed(seed)
    e = torch.randn(n, d, generator=g).bfloat16()
    c = (torch.randn(v, d, generator=g) * sigma / d ** 0.5).bfloat16()
    t = torch.randint(0, v, (n,), generator=g)
    if ignore_frac:
        t[torch.rand(n, generator=g) < ignore_frac] = -100
    E = e.float().numpy(); C = c.float().numpy(); T = t.numpy().copy(); T[T == -100] = -1
    dev = torch.device("cuda")
    ed, cd, td = e.to(dev), c.to(dev), t.to(dev)
    t0 = time.time()
    lse_l, corr = ops.forward_local(ed, cd, td, -100, 0, softcap)
    lse, loss = ops.merge_shards(lse_l[None], corr[None], td, -100)
    torch.cuda.synchronize()
    rl, rlse, rmean = O.naive_forward(E, C, T, softcap)
    valid = T != -1
    el = O.rel_err(loss.cpu().numpy(), rl)
    else_ = O.rel_err(lse.cpu().numpy()[valid], rlse[valid])
    nv = int(valid.sum())
    up = np.zeros(n, np.float32); up[valid] = 1.0 / max(nv, 1)
    upd = torch.from_numpy(up).to(dev)
    de, dc, cnt, perm = ops.backward(ed, cd, td, lse, upd, ignore_index=-100, softcap=softcap, eps=eps, vocab_sorting=sort)
    torch.cuda.synchronize()
    pm = perm.cpu().numpy() if perm is not None else None
    ce, cl, idx = O.filter_ignored(E, T)
    rde_c, rdc, st = O.lse_backward_blocked(ce, C, cl, rlse[idx].astype(np.float32), up[idx], eps=eps, perm=pm, softcap=softcap, return_stats=True)
    rde = np.zeros_like(E); rde[idx] = rde_c
    fde, fdc = O.naive_backward(E, C, T, up, softcap)
    k = cnt.cpu().tolist()
    print(f"n={n} d={d} v={v} sig={sigma} ign={ignore_frac} cap={softcap} sort={sort} eps={eps}: "
          f"loss {el:.2e} lse {else_:.2e} | dE(blk) {O.rel_err(de.float().cpu().numpy(), rde):.2e} dC(blk) {O.rel_err(dc.float().cpu().numpy(), rdc):.2e} "
          f"| dE(f64) {O.rel_err(de.float().cpu().numpy(), fde):.2e} dC(f64) {O.rel_err(dc.float().cpu().numpy(), fdc):.2e} "
          f"| gpu kept/eps/zero {k} ref eps-skip {st['skipped_epsilon']}/{st['total_tiles']} ({time.time()-t0:.1f}s)", flush=True)

if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("fwd", "all"):
        case(256, 128, 1000, sort=False, eps=0)
    if which in ("nosort", "all"):
        case(256, 128, 1000, sort=False)
        case(300, 256, 2000, sort=False, sigma=3.0)
    if which in ("sort", "all"):
        case(256, 128, 1000, sort=True)
    if which in ("ignore", "all"):
        case(512, 128, 1500, ignore_frac=0.3, sort=False)
        case(512, 128, 1500, ignore_frac=0.3, sort=True)
    if which in ("cap", "all"):
        case(256, 192, 1200, softcap=3.0, sigma=4.0, sort=True)
    if which in ("big", "all"):
        case(1024, 768, 50257, sort=True)
