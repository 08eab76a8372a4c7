"""B200-native Cut Cross-Entropy (arXiv 2411.09009).

`linear_cross_entropy` is the drop-in loss; `api` mirrors the reference package's hot-path
surface (cce_loss, lse_forward, lse_backward, ...) on CUDA tensors.  All compute runs in
libcce_b200.so (hand-written sm_100a kernels); there is no CPU fallback.
"""

from .linear_ce import linear_cross_entropy
from .ops import EPSILON_DEFAULT, BackwardStats

__all__ = ["linear_cross_entropy", "EPSILON_DEFAULT", "BackwardStats"]
__version__ = "0.1.0"
