"""paper_2009_00166_b200 -- B200-native hot path of ParIS+ exact k-NN search.

Thin Python binding (argument marshalling only) over the C ABI of
``libparis.so`` declared in ``include/paris.h``: every step of the path runs in
the library's CUDA kernels (sm_100a).  PyTorch provides device memory and
streams.  There is no CPU fallback: if the extension is missing or no CUDA
device is present, every call raises.

    sax = summarize(raw, w=16, card=256)                    # [w][n] uint8
    idx, dist = knn_exact(raw, sax, queries, k=1, w=16, card=256)
"""
from ._binding import (  # noqa: F401
    PARIS_EINVAL, PARIS_ECONFIG, PARIS_ECUDA, PARIS_ENOMEM, PARIS_MAX_K,
    ParisError, KnnConfig, Index, PARIS_INDEX_BLOCK, PARIS_INDEX_TILE, library_path, load, summarize, knn_exact,
    summarize_file, MappedRaw,
    index_build, knn_index, knn_nb, knn_approx, merge_topk, last_error, raw_bf16, paa_f16, release_workspace,
    profile_enable, profile_reset, profile_read, launch_count, version, debug_cuts, debug_half_dir, debug_read_probe, debug_set_variant, debug_gf_mma,
    debug_hfma2_probe, symbols,
)
