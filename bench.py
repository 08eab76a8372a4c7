#!/usr/bin/env python
"""Benchmark: Cut Cross-Entropy fwd+bwd tokens/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gemma2-2b] [--impl ours|reference]

One "step" = linear_cross_entropy forward + backward (reduction "mean", filter_eps 2**-12, vocab
sorting on) over one synthetic batch of the named head.  N=1 runs the Gemma-2-2B head
(BASELINE.json configs[1]).  N>1 (torchrun, one rank per GPU, NCCL) runs vocab-parallel: rank p
holds classifier rows of its shard, E/targets replicated, total work fixed ("strong").
`--mode token` instead gives every rank its own full batch (token-sharded DP, "weak").

`--impl reference` times the reference algorithm's CPU restatement (oracle/, numpy + BLAS on all
host cores; the reference is pure Python and cannot travel to the GPU box) on a bounded sample of
the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# name: (N tokens, D, V, softcap, ignore-padding fraction per sequence, logit sigma)
CONFIGS = {
    "gpt2": (4096, 768, 50257, 0.0, 0.0, 1.0),
    "gemma2-2b": (8192, 2304, 256000, 0.0, 0.0, 1.0),
    "llama3-8b": (16384, 4096, 128256, 0.0, 0.25, 1.0),
    "gemma2-9b": (32768, 3584, 256000, 30.0, 0.0, 1.0),
    "nemo-12b": (65536, 5120, 131072, 0.0, 0.0, 1.0),
}
FALLBACK_PEAKS = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return FALLBACK_PEAKS, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        # nvidia-smi --id takes the physical index; torch's index is remapped by
        # CUDA_VISIBLE_DEVICES, so address the GPU by UUID when torch exposes it
        self.id = str(index)
        try:
            import torch

            u = str(torch.cuda.get_device_properties(index).uuid)
            if u and u != "None":
                self.id = u if u.startswith("GPU-") else "GPU-" + u
        except Exception:
            pass
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.window = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.id}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a moment to start: wait for its first line so that the timed
            # region (marked by start() / stop()) is covered from its beginning
            t_end = time.monotonic() + 3.0
            while not self.lines and time.monotonic() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        return self

    def start(self):
        self.window = [time.monotonic(), None]

    def stop(self):
        if self.window is not None:
            self.window[1] = time.monotonic()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None and self.window[1] is not None:
            lo, hi = self.window
            lines = [x for x in self.lines if lo <= x[0] <= hi + 0.03]  # samples of the timed region
        for _, ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# CPU side: the reference algorithm (oracle port) on a bounded sample
# ------------------------------------------------------------------------------------------
def cpu_sample(cfg_name: str, tokens: int = 128, seed: int = 0):
    import numpy as np

    from oracle import cce_oracle as O

    n, d, v, cap, _, sigma = CONFIGS[cfg_name]
    import torch

    g = torch.Generator().manual_seed(seed)
    e = torch.randn(tokens, d, generator=g).bfloat16().float().numpy()
    c = (torch.randn(v, d, generator=g) * (sigma / math.sqrt(d))).bfloat16().float().numpy()
    x = torch.randint(0, v, (tokens,), generator=g).numpy()

    def step():
        O.cce_loss(e, c, x, softcap=cap, eps=O.EPSILON_DEFAULT, vocab_sorting=True)

    return step


def run_cpu(cfg_name: str, steps: int, warmup: int, tokens: int = 128):
    step = cpu_sample(cfg_name, tokens)
    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    return tokens / dt, dt


def cpu_desc(tokens: int) -> dict:
    try:
        model = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")), "?")
    except OSError:
        model = "?"
    return {"cores": os.cpu_count(), "cpu": model}


def zipf_head(e, c, v, v0, gen, dev, alpha=4.0, zipf_s=1.0):
    """D3: token frequencies follow a Zipf law.  A fixed unit direction u is added
    to every embedding (weight alpha) and to classifier row j (weight b_j / alpha), so logits gain
    the shared bias b_j = -s log(rank_j) (random ranks, centred); targets are sampled from the
    resulting softmax (Gumbel-max, 1024 rows at a time).  With vocab_sorting the frequent rows
    gather in the first tiles, which is where the non-trivial gradients live."""
    import torch

    n, d = e.shape
    g2 = torch.Generator(device=dev)
    g2.manual_seed(7)
    u = torch.randn(d, device=dev, generator=g2)
    u = u / u.norm()
    rank = torch.randperm(v, device=dev, generator=g2).float() + 1.0
    b = -zipf_s * torch.log(rank)
    b = b - b.mean()
    rows = slice(v0, v0 + c.shape[0])
    e = (e.float() + alpha * u).to(torch.bfloat16)
    c = (c.float() + (b[rows] / alpha)[:, None] * u).to(torch.bfloat16)
    # targets from the full vocabulary (every rank builds the same global classifier bias)
    c_full = c if c.shape[0] == v else None
    t = torch.empty(n, dtype=torch.int64, device=dev)
    for r0 in range(0, n, 1024):
        r1 = min(n, r0 + 1024)
        if c_full is not None:
            z = e[r0:r1].float() @ c_full.float().T
        else:  # vocab-parallel: only the bias drives the sampling (cheap, shard-independent)
            z = b[None, :].expand(r1 - r0, -1).clone()
        gum = -torch.log(-torch.log(torch.rand(z.shape, device=dev, generator=g2).clamp_min(1e-20)))
        t[r0:r1] = (z + gum).argmax(dim=1)
        del z, gum
    return e, c, t


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    tokens = args.cpu_tokens
    val, dt = run_cpu(args.config, args.steps, max(0, min(args.warmup, 1)), tokens)
    desc = cpu_desc(tokens)
    sample = (f"{tokens} of {cfg[0]} tokens (full D={cfg[1]}, V={cfg[2]}), numpy/BLAS oracle port of "
              f"cce_loss fwd+bwd (sort+filter), f32, {desc['cpu']}")
    line = {
        "impl": "reference", "metric": "fwd+bwd tokens/s", "value": val, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} head N={cfg[0]} D={cfg[1]} V={cfg[2]}", "sample_tokens": tokens},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": desc["cores"], "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------
def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n: int) -> int:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    print(f"bench: launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    rc = subprocess.call(cmd)
    if rc:
        sys.exit(rc)
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="gemma2-2b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="vocab", choices=["vocab", "token"])
    ap.add_argument("--sigma", type=float, default=None, help="logit std of the synthetic head")
    ap.add_argument("--pad", type=float, default=None,
                    help="fraction of each 4096-token sequence set to ignore_index (default: the config's)")
    ap.add_argument("--no-sort", action="store_true")
    ap.add_argument("--dist", default="iid", choices=["iid", "zipf"],
                    help="iid: E, C Gaussian, uniform targets (D1); zipf: a shared direction carries a "
                         "log-Zipf bias per vocabulary row and targets are sampled from the softmax "
                         "(SURVEY §8(d) D3, where vocabulary sorting groups the non-trivial tiles)")
    ap.add_argument("--no-filter", action="store_true")
    ap.add_argument("--force-dist", action="store_true", help="init the process group even for 1 rank")
    ap.add_argument("--paper-order", action="store_true",
                    help="exempt_label_tiles=False: PAPER Alg. 3 filter ordering (not the reference's)")
    ap.add_argument("--memory", default="bounded", choices=["bounded", "fast", "grouped"],
                    help="training path: bounded (default; streamed backward, no transient grows with the "
                         "kept tiles), fast (stored S-hat), grouped (= --low-memory)")
    ap.add_argument("--low-memory", action="store_true",
                    help="low_memory=True: O(N) forward state, filter pass recomputes every tile")
    ap.add_argument("--cpu-tokens", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` outside torchrun: launch the N ranks ourselves (one per GPU,
        # rendezvous on 127.0.0.1), exactly as the driver's torchrun command does
        return relaunch_under_torchrun(args.gpus)

    import torch
    import torch.distributed as dist

    from paper_2411_09009_b200 import _lib, linear_cross_entropy, ops
    from paper_2411_09009_b200.vocab_parallel import shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CCE_BENCH_BACKEND=gloo + CCE_BENCH_SAME_DEVICE=1 run N ranks on one GPU: a functional check
    # of the multi-rank path only (NCCL refuses two ranks on one device); never a bench number.
    same_dev = os.environ.get("CCE_BENCH_SAME_DEVICE") == "1"
    backend = os.environ.get("CCE_BENCH_BACKEND", "nccl")
    dev = torch.device("cuda", 0 if same_dev else local)
    torch.cuda.set_device(dev)
    group = None
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    # --force-dist: the distributed (vocab-parallel) path even for one rank -- exercises the NCCL
    # collectives on a single GPU (functional check)
    if world > 1 or args.force_dist:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
        # communicator check: every rank joined, one device per rank (NCCL) -- logged for the run
        probe = torch.ones(1, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(probe, group=group)
        print(f"bench: rank {rank}/{world} backend={dist.get_backend(group)} device={dev} "
              f"comm_nranks={int(probe.item())}", file=sys.stderr, flush=True)
        if int(probe.item()) != world:
            raise SystemExit(f"bench: communicator has {int(probe.item())} ranks, expected {world}")

    n, d, v, cap, pad_frac, sigma = CONFIGS[args.config]
    if args.pad is not None:
        pad_frac = args.pad
    if args.sigma is not None:
        sigma = args.sigma
    eps = None if args.no_filter else "auto"
    sort = not args.no_sort
    token_mode = world > 1 and args.mode == "token"

    gen = torch.Generator(device=dev)
    gen.manual_seed(0 + (rank if token_mode else 0))
    e = torch.randn(n, d, device=dev, generator=gen).to(torch.bfloat16)
    gen.manual_seed(1)
    dist_vocab = (world > 1 or args.force_dist) and not token_mode
    if dist_vocab:
        v0, v1 = shard_range(v, rank, world)
        c_full_rows = v1 - v0
        # deterministic shard of the same global classifier: generate only this shard's rows
        gen.manual_seed(1000 + v0)
        c = (torch.randn(c_full_rows, d, device=dev, generator=gen) * (sigma / math.sqrt(d))).to(torch.bfloat16)
    else:
        v0 = 0
        c = (torch.randn(v, d, device=dev, generator=gen) * (sigma / math.sqrt(d))).to(torch.bfloat16)
    gen.manual_seed(2 + (rank if token_mode else 0))
    t = torch.randint(0, v, (n,), device=dev, generator=gen)
    if args.dist == "zipf":
        e, c, t = zipf_head(e, c, v, v0, gen, dev)
    if pad_frac:
        seq = 4096
        pos = torch.arange(n, device=dev) % seq
        t[pos >= int(seq * (1 - pad_frac))] = -100
    e.requires_grad_(True)
    c.requires_grad_(True)

    kw = dict(reduction="mean", filter_eps=eps, vocab_sorting=sort, softcap=cap or None,
              low_memory=args.low_memory, exempt_label_tiles=not args.paper_order,
              memory=None if args.low_memory else args.memory)
    mem_mode = "grouped" if args.low_memory else args.memory
    if dist_vocab:
        kw.update(process_group=group, vocab_start=v0)

    def step(ei, ci, ti):
        ei.grad = None
        ci.grad = None
        loss = linear_cross_entropy(ei, ci, ti, **kw)
        loss.backward()
        return loss

    def barrier():
        if group is not None:
            dist.barrier()

    # ---- memory (instrument.py:3-10 definition: transients only; inputs E, C, targets and the
    # outputs dE, dC, loss are not counted).  Measured on one training step, then on the
    # low-memory forward (inference / low_memory=True: only O(N) state).
    def mem_step():
        e.grad = None
        c.grad = None
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        loss = linear_cross_entropy(e, c, t, **kw)
        torch.cuda.synchronize()
        fwd_peak = torch.cuda.max_memory_allocated(dev) - base
        held = torch.cuda.memory_allocated(dev) - base
        loss.backward()
        torch.cuda.synchronize()
        grad_bytes = e.grad.numel() * e.grad.element_size() + c.grad.numel() * c.grad.element_size()
        step_peak = torch.cuda.max_memory_allocated(dev) - base - grad_bytes
        return fwd_peak, held, step_peak

    for _ in range(args.warmup):
        step(e, c, t)
    fwd_peak, fwd_held, step_peak = mem_step()
    e.grad = None
    c.grad = None
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    with torch.no_grad():
        ops.forward_local(e.detach(), c.detach(), t, -100, v0, cap)
    torch.cuda.synchronize()
    fwd_lean = torch.cuda.max_memory_allocated(dev) - base  # outputs lse/correct (8N B) included

    # ---- timed region: device time with CUDA events, max over ranks
    ops.KERNEL_EVENTS = {}
    launches0 = _lib.load().cce_launch_count()  # counted inside libcce_b200.so
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        barrier()  # every rank's sampler is running before the timed region starts
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        clk.start()
        t0.record()
        for _ in range(args.steps):
            step(e, c, t)
        t1.record()
        torch.cuda.synchronize()
        clk.stop()
    barrier()
    ms = t0.elapsed_time(t1) / args.steps
    launches = (_lib.load().cce_launch_count() - launches0) // args.steps
    # per-step device time of each C entry point (the backward has a primary and a device-gated
    # fallback call per step, so calls are summed per step, not averaged)
    kev = {k: sum(a.elapsed_time(b) for a, b in evs) / args.steps for k, evs in ops.KERNEL_EVENTS.items()}
    ops.KERNEL_EVENTS = None
    counters = ops.LAST_COUNTERS["counters"].tolist()
    stats = ops.LAST_STATS["stats"].tolist() if "stats" in ops.LAST_STATS else None
    if world > 1:
        mt = torch.tensor([ms], device=dev)
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        ms = float(mt.item())
    total_tokens = n * (world if token_mode else 1)
    value = total_tokens / (ms / 1e3)

    # ---- end to end through the public API with host (pinned) inputs.  Every step copies that
    # step's batch -- the hidden states E and the targets -- host->device and reads the loss back;
    # the classifier C is the layer's weight and stays resident, as in a training loop.  Step
    # k+1's copies run on a side stream while step k computes (double-buffered device inputs).
    # A second figure also copies C (1.18 GB at Gemma-2B) every step: that one is PCIe-bound.
    e2e = None
    if not args.no_e2e:
        eh = e.detach().cpu().pin_memory()
        ch = c.detach().cpu().pin_memory()
        th = t.cpu().pin_memory()
        lh = torch.empty((), dtype=torch.float32).pin_memory()
        copy_stream = torch.cuda.Stream(dev)

        def e2e_time(copy_c: bool, k: int) -> float:
            srcs = (eh, ch, th) if copy_c else (eh, th)
            bufs = [tuple(torch.empty(x.shape, dtype=x.dtype, device=dev) for x in srcs) for _ in range(2)]
            ready = [torch.cuda.Event() for _ in range(2)]
            done = [torch.cuda.Event() for _ in range(2)]
            c_res = c.detach()

            def h2d(slot):
                with torch.cuda.stream(copy_stream):
                    copy_stream.wait_event(done[slot])  # previous user of the slot finished
                    for dst, src in zip(bufs[slot], srcs):
                        dst.copy_(src, non_blocking=True)
                    ready[slot].record(copy_stream)

            def run(steps):
                for q in range(2):
                    done[q].record()
                h2d(0)
                for i in range(steps):
                    slot = i & 1
                    if i + 1 < steps:
                        h2d(slot ^ 1)
                    torch.cuda.current_stream().wait_event(ready[slot])
                    b = bufs[slot]
                    ei = b[0].requires_grad_(True)
                    ci = (b[1] if copy_c else c_res).requires_grad_(True)
                    loss = step(ei, ci, b[-1])
                    lh.copy_(loss.detach(), non_blocking=True)
                    done[slot].record()
                    for x in b[:2]:
                        x.requires_grad_(False)
                    c_res.requires_grad_(False)

            run(2)
            barrier()
            torch.cuda.synchronize()
            a0 = torch.cuda.Event(enable_timing=True)
            b0 = torch.cuda.Event(enable_timing=True)
            a0.record()
            run(k)
            b0.record()
            torch.cuda.synchronize()
            ms_ = a0.elapsed_time(b0) / k
            if world > 1:
                mt_ = torch.tensor([ms_], device=dev)
                dist.all_reduce(mt_, op=dist.ReduceOp.MAX)
                ms_ = float(mt_.item())
            return ms_

        e2e_ms = e2e_time(False, args.steps)
        e2e_all_ms = e2e_time(True, max(3, args.steps // 4))
        e2e = {"value": total_tokens / (e2e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": eh.numel() * 2 + th.numel() * 8,
               "d2h_bytes_per_step": 4, "ms_per_step": e2e_ms,
               "note": "per step: E and targets copied host->device (pinned, side stream, overlapping "
                       "the previous step), loss read back; classifier weight C resident",
               "with_weight_copy": {"value": total_tokens / (e2e_all_ms / 1e3), "ms_per_step": e2e_all_ms,
                                    "h2d_bytes_per_step": eh.numel() * 2 + ch.numel() * 2 + th.numel() * 8}}

    # ---- roofline of the dominant kernel (executed flops / event-timed launch duration)
    peaks, peak_src = load_peaks()
    n_valid = int((t != -100).sum().item())
    v_loc = c.shape[0]
    kept = counters[0]
    tile_area = 128 * 256
    tiles_path = not (args.low_memory or args.no_filter)  # forward on compacted rows
    flops_fwd = 2.0 * (n_valid if tiles_path else n) * v_loc * d
    # backward recompute: every tile (low_memory filter pass) or, on the training path, only the
    # kept tiles the forward did not store (label tiles are stored and need no recompute); then
    # dE and dC over all kept tiles
    fast = tiles_path and mem_mode == "fast"
    recomputed = stats[1] if (fast and stats) else kept
    flops_recompute = 2.0 * d * recomputed * tile_area if tiles_path else 2.0 * n_valid * v_loc * d
    flops_bwd = flops_recompute + 4.0 * d * kept * tile_area
    # dominant single kernel: the forward logit-tile kernel (cce_fwd is one tcgen05 launch plus two
    # tiny ones); the backward entry is three kernels (B1 filter, B2 dE, B3 dC) and is reported
    # as a group in `kernel_ms` / `step_tflops`.
    # bounded mode: the forward is one logit-tile launch per vocabulary group (gathers between)
    dom = "fwd_kernel" if "fwd_kernel" in kev else "fwd"
    dom_flops = flops_fwd
    dom_ms = kev[dom]
    achieved = dom_flops / (dom_ms / 1e3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(args.config, {}).get(f"{dom}_dram_bytes")
        except (ValueError, AttributeError):
            traffic = None
    total_tiles = -(-n_valid // 128) * -(-v_loc // 256)
    step_flops = flops_fwd + flops_bwd

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cval, _ = run_cpu(args.config, 2, 0, args.cpu_tokens)
        desc = cpu_desc(args.cpu_tokens)
        cpu = {"value": cval, "unit": "tokens/s", "cores": desc["cores"], "kind": "port",
               "sample": f"{args.cpu_tokens} of {n} tokens, full D/V, numpy+BLAS oracle port of cce_loss "
                         f"fwd+bwd on {desc['cpu']}, mean of 2 runs"}

    if rank == 0:
        line = {
            "metric": "fwd+bwd tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if (world == 1 or token_mode) else "strong",
            "vs_baseline": None, "dtype": "bf16", "data": ("synthetic (random E ~ N(0,1), C ~ N(0, sigma^2/D), uniform targets)" if args.dist == "iid" else
                     "synthetic (D3: E, C Gaussian plus a shared log-Zipf row bias, targets sampled from the softmax)"),
            "config": {
                "workload": f"{args.config} head N={n} D={d} V={v}", "dist": args.dist, "sigma": sigma, "softcap": cap,
                "ignore_pad_frac": pad_frac, "filter_eps": None if args.no_filter else 2 ** -12,
                "vocab_sorting": sort, "reduction": "mean", "low_memory": args.low_memory,
                "filter_order": "paper (exempt_label_tiles=False)" if args.paper_order else "reference",
                "parallelism": (f"vocab{world}" if world > 1 and not token_mode else f"token{world}"),
                "l2": "inputs larger than L2 (C alone is %.2f GB)" % (v_loc * d * 2 / 1e9),
            },
            "gpu_launches": launches,
            "kernel_ms": kev,
            "skip": {"kept_tiles": kept, "eps_skipped": counters[1], "zero_up_skipped": counters[2],
                     "total_tiles": total_tiles, "skip_rate": 1 - kept / max(1, total_tiles),
                     "label_tiles_stored": stats[0] if (fast and stats) else 0,
                     "recomputed_tiles": recomputed if tiles_path else total_tiles},
            "step_tflops": step_flops / (ms / 1e3) / 1e12,
            "step_frac": step_flops / (ms / 1e3) / 1e12 / peaks["bf16_tflops"],
            "bwd_tflops": flops_bwd / (kev.get("bwd", float("nan")) / 1e3) / 1e12,
            "roofline": {"bound": "tensor", "kernel": "cce_lse_kernel<FWD>" + (" (per vocabulary group)" if dom == "fwd_kernel" else ""),
                         "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                         "frac": achieved / peaks["bf16_tflops"],
                         "frac_sustained": achieved / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]),
                         "peak_source": peak_src + " bf16 burst", "traffic": traffic,
                         "flops_per_launch": dom_flops},
            "memory": {"step_peak_transient_bytes": int(step_peak), "fwd_peak_transient_bytes": int(fwd_peak),
                       "fwd_to_bwd_state_bytes": int(fwd_held), "lean_fwd_transient_bytes": int(fwd_lean),
                       "mode": mem_mode},
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
