"""paper_2307_12059_b200 -- B200-native TransE completion join (arXiv 2307.12059).

The product is libkgc.so (C ABI in include/kgc.h, CUDA kernels for sm_100a in
csrc/); ``kgc`` is its thin ctypes binding.  No CPU fallback exists.
"""
from .kgc import (Join, KgcError, TRIPLET_DTYPE, kgc_abi_version, kgc_create, kgc_default_options,  # noqa: F401
                  kgc_destroy, kgc_inspect, kgc_join, kgc_last_error, kgc_results, kgc_set_stream,
                  kgc_shard_range, kgc_stats, load_library)
