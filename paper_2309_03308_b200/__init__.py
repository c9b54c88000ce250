"""B200-native (sm_100a) hot path of arXiv 2309.03308: batched KSG-MI / Pearson point
pairs of a 3D ensemble field, reduced to per-region-pair maxima.

The product is libcorr.so (C ABI in include/corr.h, CUDA kernels in csrc/); this
package holds its thin binding (``binding``), the seeded input generator (``synth``)
and the multi-GPU sharding helpers (``dist``).
"""
from .binding import (CORR_F_ABS, CORR_F_KSG_PLUS1, CORR_KSG, CORR_PEARSON, CorrError, Field,  # noqa: F401
                      corr_check, corr_eval_pairs, corr_field_aggregate, corr_field_create, corr_field_destroy, corr_field_info,
                      corr_ksg_debug, corr_region_max)
