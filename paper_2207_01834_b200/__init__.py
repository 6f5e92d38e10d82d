"""B200-native BDL-tree hot path (kNN_L + BuildvEB_S) of arxiv 2207.01834 (ParGeo).

The product is the C-ABI library _lib/libgkbdl.so (include/gk_bdl.h, CUDA for
sm_100a); this package is its Python host mirror.
"""
from .bdltree import (BDLTree, GpuError, KnnCounters, MAX_K, NO_POINT, OBJECT_MEDIAN, SPATIAL_MEDIAN,  # noqa: F401
                      gen_mixture, gen_uniform, gen_walk, l2_read_gbs, lib, sample_without_replacement)
from .configs import CONFIGS, make_inputs  # noqa: F401
