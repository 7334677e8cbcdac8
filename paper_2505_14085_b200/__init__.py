"""B200-native CE-LSLM cloud->edge KV-reuse path (arXiv 2505.14085).

Stage 1  layer-alignment map + projection of cloud K/V into edge head geometry
Stage 2  representation compression (gather, int8/int4 quantise, pack)
Stage 3  edge decode attention over the reused, dequantised KV (Eq. 5 merge)

Kernels: paper_2505_14085_b200/csrc (sm_100a), C ABI: include/ekv_capi.h,
C++ mirror of the reference interface: include/edgekv_b200.hpp.
"""
from .capi import EkvError, load  # noqa: F401

__version__ = "0.1.0"
