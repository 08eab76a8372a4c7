"""PAPER.md Table 1 (tab:perf) on one B200: peak memory and time of the loss, its gradient and
both, for CCE and the paper's comparators, at the Gemma-2-2B head shape (N=8192, D=2304,
V=256000, bf16).

Inputs are synthetic (E ~ N(0,1), C ~ N(0, 1/D): logit std 1), not the Gemma-2 embeddings of the
paper, so gradient-filter skip rates differ from the paper's.  Memory = peak allocation above the
inputs, gradient outputs included (the paper's convention; "lower bound" = dE + dC).  Times are
medians of CUDA-event-timed repetitions.  Liger is the installed liger_kernel (Triton); it is a
comparator only, never part of this package's path.
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

from paper_2411_09009_b200 import linear_cross_entropy

N, D, V = 8192, 2304, 256000
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
E = torch.randn(N, D, device=dev, generator=g).bfloat16()
C = (torch.randn(V, D, device=dev, generator=g) / math.sqrt(D)).bfloat16()
T = torch.randint(0, V, (N,), device=dev, generator=g)


def baseline(e, c, t):
    return F.cross_entropy((e @ c.T).float(), t)


compiled = torch.compile(baseline)


def chunked8(e, c, t):  # torchtune-style: 8 token chunks, logits upcast per chunk
    total = 0.0
    for ec, tc in zip(e.chunk(8), t.chunk(8)):
        total = total + F.cross_entropy((ec @ c.T).float(), tc, reduction="sum")
    return total / t.numel()


def liger(e, c, t):
    from liger_kernel.ops.fused_linear_cross_entropy import LigerFusedLinearCrossEntropyFunction

    return LigerFusedLinearCrossEntropyFunction.apply(e, c, t)[0]


METHODS = {
    "CCE (ours)": lambda e, c, t: linear_cross_entropy(e, c, t),
    "CCE memory=fast": lambda e, c, t: linear_cross_entropy(e, c, t, memory="fast"),
    "CCE low_memory": lambda e, c, t: linear_cross_entropy(e, c, t, low_memory=True),
    "CCE (no vocab sorting)": lambda e, c, t: linear_cross_entropy(e, c, t, vocab_sorting=False),
    "CCE (no grad filter)": lambda e, c, t: linear_cross_entropy(e, c, t, filter_eps=None),
    "Liger": liger,
    "torchtune-style (8 chunks)": chunked8,
    "torch.compile": compiled,
    "Baseline (torch)": baseline,
}


def measure(fn, phase, reps=10):
    def once():
        e = E.detach().requires_grad_(phase != "loss")
        c = C.detach().requires_grad_(phase != "loss")
        if phase == "loss":
            with torch.no_grad():
                return fn(e, c, T), None
        loss = fn(e, c, T)
        return loss, (e, c)

    for _ in range(2):
        out = once()
        if phase != "loss":
            out[0].backward()
        del out
    torch.cuda.synchronize()
    times = []
    peak = 0
    for _ in range(reps):
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        if phase == "grad":
            loss, keep = once()
            torch.cuda.synchronize()
            base = torch.cuda.memory_allocated()
            torch.cuda.reset_peak_memory_stats()
            a.record()
            loss.backward()
            b.record()
        else:
            a.record()
            loss, keep = once()
            if phase == "both":
                loss.backward()
            b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        peak = max(peak, torch.cuda.max_memory_allocated() - base)
        del loss, keep
    times.sort()
    return peak / 2**20, times[len(times) // 2]


rows = []
for name, fn in METHODS.items():
    row = {"method": name}
    for phase in ("loss", "grad", "both"):
        try:
            mem, ms = measure(fn, phase)
            row[phase] = {"mem_mb": round(mem, 1), "ms": round(ms, 3)}
        except Exception as exc:  # a comparator that cannot run here is reported, not fatal
            row[phase] = {"error": f"{type(exc).__name__}: {str(exc)[:120]}"}
        torch.cuda.empty_cache()
    rows.append(row)
    print(json.dumps(row), flush=True)

lb = (N * D + V * D) * 2 / 2**20
lines = ["| Method | Loss mem | Loss time | Grad mem | Grad time | Loss+grad mem | Loss+grad time |",
         "|---|---|---|---|---|---|---|",
         f"| Lower bound (dE + dC) | 0 | | {lb:.0f} MB | | {lb:.0f} MB | |"]
for r in rows:
    cells = []
    for ph in ("loss", "grad", "both"):
        x = r[ph]
        cells += ([f"{x['mem_mb']:.0f} MB", f"{x['ms']:.2f} ms"] if "ms" in x else ["n/a", "n/a"])
    lines.append(f"| {r['method']} | " + " | ".join(cells) + " |")
print("\n".join(lines))
