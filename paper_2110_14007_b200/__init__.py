"""B200-native exact kNN / LOF outlier scoring (TOD, arXiv 2110.14007 hot path).

The compute path is libtod.so (CUDA sm_100a, C ABI in include/tod.h); this
package only loads it and marshals arguments (tod.py) and shards rows across
processes (dist.py).  It never imports the CPU oracle (oracle/), and it has no
CPU fallback.
"""
from .tod import (Context, KnnResult, TodError, load_library, header_symbols, LIB_PATH,  # noqa: F401
                  F_NO_CERTIFY, F_TIMING, F_PASS1_V1, F_MAIN_1SM, FORMATS, MAX_K,
                  comm_id_create, shard_rows, workspace_size)

from . import detectors  # noqa: F401,E402  (PyOD-style fit/decision_scores_/labels_)

__all__ = ["detectors", "Context", "KnnResult", "TodError", "load_library", "header_symbols", "LIB_PATH",
           "F_NO_CERTIFY", "F_TIMING", "F_PASS1_V1", "F_MAIN_1SM", "FORMATS", "MAX_K",
           "comm_id_create", "shard_rows", "workspace_size"]
