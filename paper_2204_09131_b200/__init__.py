"""paper_2204_09131_b200 — B200-native (sm_100a) hot path of iSYCOS (arXiv 2204.09131).

Batched KSG window mutual information and the SYCOS_TD / SYCOS_BU / noise-pruning search that
consumes it, behind the C ABI of libisycos.so (include/isycos.h).  This package is the thin
Python binding (ctypes, argument marshalling only) plus the torch.distributed sharding helpers
(``dist``).  There is no CPU fallback: if libisycos.so is missing the calls raise.
"""
from ._capi import (  # noqa: F401
    EXPORTS,
    IsycosError,
    isycos_abi_version,
    isycos_last_error,
    isycos_mi_batch,
    isycos_mi_batch_ex,
    isycos_merge_windows,
    isycos_release_cache,
    isycos_search,
    lib,
    search_workload,
)

__all__ = ["isycos_mi_batch", "isycos_mi_batch_ex", "isycos_search", "isycos_last_error",
           "isycos_abi_version", "isycos_release_cache", "isycos_merge_windows", "IsycosError", "search_workload"]
