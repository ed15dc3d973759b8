"""paper_2406_10938_b200 — B200-native (sm_100a) DET-LSH index build and
c^2-k-ANN query (arxiv 2406.10938), behind the reference's build/query API.

The compute path is the in-tree CUDA library ``libdetlsh_b200.so`` reached
through the C ABI in ``include/detlsh_b200.h``; this package is the thin
host-side mirror of the reference interface (see api.py).
"""
from .api import (  # noqa: F401
    SAMPLE_GPU,
    SAMPLE_REFERENCE,
    BatchResult,
    DerivedParams,
    DetIndex,
    LshParams,
    QueryResult,
    TreeExport,
    brute_force_knn,
    brute_force_knn_device,
    build_det_only_index,
    build_index,
    build_index_with_family,
    build_sharded_index,
    ck_ann_sharded,
    ck_ann_sharded_device,
    ShardedIndex,
    rc_ann,
    rc_ann_batch,
    read_vectors_device,
    vectors_shape,
    build_tree,
    candidate_budget,
    chi2_cdf,
    chi2_quantile,
    ck_ann,
    ck_ann_batch,
    ck_ann_device,
    derive_params,
    device_count,
    encode_dataset,
    estimate_rmin,
    range_query_exact,
    range_query_optimized,
    merge_topk_device,
    mix_seed,
    project_dataset,
    query_check,
    sample_hash_family,
    select_breakpoints,
)
from ._lib import FormatError, LIB_PATH, header_symbols, load  # noqa: F401

__version__ = "0.1.0"
