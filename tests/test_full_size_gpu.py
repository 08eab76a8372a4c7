"""Full-size parity at BASELINE.json's headline shape (Gemma-2-2B head: N=8192, D=2304, V=256000).

The f64 CPU oracle cannot run this size inside a test, so the reference here is a chunked plain
PyTorch fp32 computation on the same bf16-rounded inputs (fp32 logits, exact softmax, exact
gradients).  Tolerances: loss / lse max-norm rel <= 1e-3; unfiltered gradients
<= 1e-2; the filtered default path (eps = 2**-12, vocab sorting) against the exact gradient
<= 3e-2 (the filtering error itself, SURVEY App. B.2 measured 1.9e-2 on these logits).
"""

import math

import numpy as np
import pytest
import torch

from oracle import cce_oracle as O

pytestmark = pytest.mark.gpu

N, D, V = 8192, 2304, 256000


def _torch_reference(e, c, t, chunk=1024):
    """fp32 loss / lse per token and exact dE, dC for reduction='mean'."""
    ef, cf = e.float(), c.float()
    n_valid = int((t != -100).sum())
    loss = torch.empty(N, device=e.device)
    lse = torch.empty(N, device=e.device)
    de = torch.empty(N, D, device=e.device)
    dc = torch.zeros(V, D, device=e.device)
    for i0 in range(0, N, chunk):
        z = ef[i0:i0 + chunk] @ cf.T
        l = torch.logsumexp(z, dim=1)
        tt = t[i0:i0 + chunk]
        loss[i0:i0 + chunk] = l - z.gather(1, tt.clamp_min(0)[:, None])[:, 0]
        lse[i0:i0 + chunk] = l
        g = torch.exp(z - l[:, None])
        g[torch.arange(len(tt), device=e.device), tt] -= 1.0
        g /= n_valid
        de[i0:i0 + chunk] = g @ cf
        dc += g.T @ ef[i0:i0 + chunk]
        del z, g
    return loss, lse, de, dc


def test_gemma2b_head_full_size(cuda_device):
    from paper_2411_09009_b200 import linear_cross_entropy, ops

    torch.backends.cuda.matmul.allow_tf32 = False
    gen = torch.Generator(device="cuda").manual_seed(0)
    e = torch.randn(N, D, device="cuda", generator=gen).bfloat16()
    c = (torch.randn(V, D, device="cuda", generator=gen) / math.sqrt(D)).bfloat16()
    t = torch.randint(0, V, (N,), device="cuda", generator=gen)
    ref_loss, ref_lse, ref_de, ref_dc = _torch_reference(e, c, t)
    ref_mean = float(ref_loss.mean())
    results = {}
    for name, kw in (("unfiltered", dict(filter_eps=None)), ("default", dict())):
        ei = e.clone().requires_grad_(True)
        ci = c.clone().requires_grad_(True)
        out = linear_cross_entropy(ei, ci, t, **kw)
        out.backward()
        torch.cuda.synchronize()
        assert abs(out.item() - ref_mean) <= 1e-3 * abs(ref_mean), (name, out.item(), ref_mean)
        err_e = O.rel_err(ei.grad.float().cpu().numpy(), ref_de.cpu().numpy())
        err_c = O.rel_err(ci.grad.float().cpu().numpy(), ref_dc.cpu().numpy())
        results[name] = (err_e, err_c, ops.LAST_COUNTERS["counters"].cpu().tolist())
    print(f"full-size parity (dE rel, dC rel, tile counters): {results}")
    assert results["unfiltered"][0] < 1e-2 and results["unfiltered"][1] < 1e-2, results
    assert results["default"][0] < 3e-2 and results["default"][1] < 3e-2, results
    kept, eps_skipped, zero = results["default"][2]
    assert kept + eps_skipped + zero == (N // 128) * (V // 256) and eps_skipped > 0
    # per-token loss / lse at full size (forward only)
    lse_l, corr = ops.forward_local(e, c, t, -100)
    lse, loss = ops.merge_shards(lse_l[None], corr[None], t, -100)
    assert float((lse - ref_lse).abs().max()) <= 1e-3 * float(ref_lse.abs().max())
    assert float((loss - ref_loss).abs().max()) <= 1e-3 * max(1.0, float(ref_loss.abs().max()))
