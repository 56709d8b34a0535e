"""StragglAR (arXiv 2505.23523) straggler-aware AllReduce for B200 (sm_100a).

The product is ``libstragglar.so`` (C ABI in ``include/stragglar.h``); this
package holds its CUDA/C++ sources (``csrc/``), the in-tree build
(``build.py``), the ctypes binding (``stragglar.py``), the multi-process
handle exchange over torch.distributed (``dist.py``) and the seeded input
generators (``inputs.py``).
"""
__all__ = ["stragglar", "dist", "inputs", "build"]
