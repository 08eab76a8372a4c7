"""Time the in-place row unpermutation (cce_unpermute_rows) at Gemma-2B's classifier shape on a
random order: CUDA events over REPS calls (each call re-permutes the rows it left)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_09009_b200 import _lib, ops  # noqa: E402

v, d = int(os.environ.get("V", 256000)), int(os.environ.get("D", 2304))
reps = int(os.environ.get("REPS", 20))
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
perm = torch.randperm(v, device="cuda", generator=g).to(torch.int32)
inv = torch.empty_like(perm)
inv[perm.long()] = torch.arange(v, dtype=torch.int32, device="cuda")
x = torch.randn(v, d, device="cuda", generator=g).bfloat16()
ws_bytes = lib.cce_bwd_stream_workspace_bytes(1, d, v, 512)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")


def run():
    _lib.check(lib.cce_unpermute_rows(ops._p(x), ops._p(perm), ops._p(inv), v, d, ops._p(ws), ws_bytes,
                                      ops._stream(x.device)), "cce_unpermute_rows")


for _ in range(3):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    run()
b.record()
torch.cuda.synchronize()
print(f"unpermute v={v} d={d}: {a.elapsed_time(b) / reps:.3f} ms ({os.environ.get('CCE_LIB', 'default')})")
