"""Per-kernel breakdown of one default training step at the Gemma-2-2B head (device times from a
torch.profiler trace of 3 steps, median per kernel), with algorithmic flops / bytes per kernel and
the fraction of the measured peaks (MEASURED_PEAKS.json).  Writes markdown to stdout."""
import json, math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2411_09009_b200 import linear_cross_entropy, ops

import bench

CFG = os.environ.get("BREAKDOWN_CONFIG", "gemma2-2b")
N, D, V, CAP, PAD, SIGMA = bench.CONFIGS[CFG]
LOW = os.environ.get("BREAKDOWN_LOW", "0") == "1"  # low_memory=True (vocabulary groups)
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
e = torch.randn(N, D, device=dev, generator=g).bfloat16().requires_grad_(True)
c = (torch.randn(V, D, device=dev, generator=g) * SIGMA / math.sqrt(D)).bfloat16().requires_grad_(True)
t = torch.randint(0, V, (N,), device=dev, generator=g)
if os.environ.get("BREAKDOWN_DIST", "iid") == "zipf":  # SURVEY D3 (bench.zipf_head)
    e, c, t = bench.zipf_head(e.detach(), c.detach(), V, 0, g, dev)
    e.requires_grad_(True)
    c.requires_grad_(True)


def step():
    e.grad = c.grad = None
    linear_cross_entropy(e, c, t, softcap=CAP or None, low_memory=LOW,
                         exempt_label_tiles=os.environ.get("BREAKDOWN_PAPER", "0") != "1").backward()


for _ in range(4):
    step()
torch.cuda.synchronize()
steps = 3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
kept = int(ops.LAST_COUNTERS["counters"][0])
recomputed = kept if LOW else int(ops.LAST_STATS["stats"][1])  # default: label tiles stored by the forward
evs = sorted([x for x in prof.events() if x.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda x: x.time_range.start)
span = (evs[-1].time_range.end - evs[0].time_range.start) / steps / 1e3
# Exclusive time: a kernel is charged only for the part of its interval not already covered by
# kernels that started earlier.  With programmatic dependent launch a kernel starts while its
# predecessor drains and waits at entry; with the label S-hat side stream two kernels overlap.
per = {}
covered = None
for x in evs:
    a, b = x.time_range.start, x.time_range.end
    lo = a if covered is None else max(a, covered)
    per.setdefault(x.name, []).append(max(0, b - lo) / 1e3)
    covered = b if covered is None else max(covered, b)
peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))) \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else \
    {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
tile = 128 * 256
work = {  # name fragment -> (flops, bytes) per step (algorithmic)
    "cce_lse_kernel<0": (2.0 * N * V * D, None),
    "cce_lse_kernel<2": (2.0 * D * recomputed * tile, None),
    "label_shat_kernel": (None, (kept - recomputed) * tile * 4.0),
    "cce_de_kernel": (2.0 * D * kept * tile, None),
    "cce_dc_kernel": (2.0 * D * kept * tile, None),
    "sort_key_kernel": (None, V * D * 2.0),
    "gather_rows_kernel": (None, 2 * (V + N) * D * 2.0),
    "decide_tiles_kernel": (None, (N // 128) * (V // 256) * 512.0),
}
rows = []
for name, ds in per.items():
    ms = sum(ds) / steps
    short = name.split("(")[0].replace("void ", "").replace("cce::", "")
    flops = byts = None
    for k, (f, b) in work.items():
        if k in name:
            flops, byts = f, b
    rows.append((ms, short, flops, byts))
rows.sort(reverse=True)
print(f"{CFG} head N={N} D={D} V={V}, {'low_memory=True' if LOW else 'default path'}, {steps} steps: {span:.2f} ms/step, kept tiles {kept} of "
      f"{(N // 128) * (V // 256)} ({kept - recomputed} stored by the forward, {recomputed} recomputed); peaks: {peaks['bf16_tflops']} TFLOP/s bf16, {peaks['hbm_gbs']} GB/s\n")
print("| kernel | ms/step (exclusive) | share | achieved | of peak |")
print("|---|---|---|---|---|")
busy = 0.0
for ms, short, f, b in rows:
    busy += ms
    if ms < 0.004:
        continue
    ach = frac = ""
    if ms < 0.05:  # gated-off fallback launches and tiny kernels: no meaningful rate
        f = b = None
    if f:
        ach = f"{f / (ms / 1e3) / 1e12:.0f} TFLOP/s"
        frac = f"{f / (ms / 1e3) / 1e12 / peaks['bf16_tflops']:.0%}"
    elif b:
        ach = f"{b / (ms / 1e3) / 1e9:.0f} GB/s"
        frac = f"{b / (ms / 1e3) / 1e9 / peaks['hbm_gbs']:.0%}"
    print(f"| `{short[:60]}` | {ms:.3f} | {ms / span:.1%} | {ach} | {frac} |")
print(f"| (all kernels) | {busy:.3f} | {busy / span:.1%} | | |")
print(f"| (gaps between kernels) | {span - busy:.3f} | {(span - busy) / span:.1%} | | |")
