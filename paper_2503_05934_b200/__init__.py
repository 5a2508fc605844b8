"""netsort-b200: merge sort and quick sort over int32 and int64 keys whose recursion
bottoms out in fixed sorting networks (arXiv 2503.05934), rebuilt for B200
(sm_100a).  The compute lives in lib/libnetsort_b200.so behind the C ABI
include/netsort_b200.h; this package is the Python host layer over it."""
from ._lib import NetsortError, build, lib  # noqa: F401
from .api import (  # noqa: F401
    Algorithm, DispatchStats, argsort, NetworkConfig, SortVariant, algorithm_name, base_case_applies,
    bundled_variants, classic_config, classical_merge_sort, classical_quick_sort,
    config_registry, count_inversions, find_config, kMaxNetworkWidth, kMinNetworkWidth,
    hoare_partition, leaf_width, make_fixed_config, median_of_three, make_varsort_config, merge, merge_sort_dispatch_stats,
    multiset_digest, network,
    optimized_merge_sort, optimized_quick_sort, quick_sort_traced, release_scratch, run_variant,
    segmented_sort, sort_host_async, sort_pairs, sort_small_batch, generate, generate_batch)
