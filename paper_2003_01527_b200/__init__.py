"""paper_2003_01527_b200 — B200-native GSM (Gunrock Subgraph Matching, arXiv 2003.01527) hot path.

The product is libgsm.so (C ABI in include/gsm.h, sm_100a kernels in csrc/);
:mod:`.gsm` is the thin ctypes binding and :mod:`.multigpu` the root-sharded
multi-GPU driver (torch.distributed over NCCL).  There is no CPU fallback.
"""
from . import gsm  # noqa: F401
from .gsm import (GSM_FLAG_NO_SYMMETRY, GSM_FLAG_PROFILE, GSM_FLAG_UNIQUE, GSM_MODE_COUNT,  # noqa: F401
                  GSM_MODE_ENUMERATE, GsmError, gsm_free, gsm_graph_info, gsm_last_error, gsm_load_graph,
                  gsm_match, gsm_plan_query, gsm_result_copy_rows, gsm_result_free)

__all__ = ["gsm", "gsm_load_graph", "gsm_match", "gsm_free", "gsm_result_free", "gsm_result_copy_rows",
           "gsm_graph_info", "gsm_plan_query", "gsm_last_error", "GsmError", "GSM_MODE_COUNT", "GSM_MODE_ENUMERATE",
           "GSM_FLAG_UNIQUE", "GSM_FLAG_NO_SYMMETRY", "GSM_FLAG_PROFILE"]
