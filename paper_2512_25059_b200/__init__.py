"""paper_2512_25059_b200 -- B200-native hot path of R²CCL (arXiv 2512.25059):
a fault-tolerant chunked multi-channel ring allreduce over NVLink 5 peer
mappings, with per-chunk completion flags, DMA-buffer rollback, failover
chains, R²CCL-Balance and three-point triangulation.

The product is the C-ABI library libr2ccl.so (include/r2ccl.h); this
package only builds it (build.py) and binds it (r2ccl.py, torch_api.py).
"""
from . import r2ccl  # noqa: F401

__all__ = ["r2ccl"]
