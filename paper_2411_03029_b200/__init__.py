"""B200-native tensor butterfly (arXiv 2411.03029) — construction and apply of
the compressed oscillatory integral operator on sm_100a.

The compute lives in ``libtbf_b200.so`` (hand-written CUDA + C++ runtime, C ABI
in ``include/oiobf_b200.h``); this package is the thin host binding.  Importing
it does not touch the GPU; the first compute call loads the library and fails
loudly if it (or a Blackwell device) is missing — there is no CPU fallback.
"""
from .configs import (CONFIGS, BY_NAME, Config, KernelSpec, dft, green_cubes, green_plates, level_rule, nudft,  # noqa
                      radon2d, radon3d)
from .butterfly import (ColumnID, ProxyStrategy, TensorButterfly, column_id, column_id_batch, dense_rows,  # noqa
                        derive_seed, mode_product_blockdiag, select_proxies, select_proxies_count, subtensor_at,
                        tbf_construct, tbf_contract, tbf_error_estimate, tbf_load, tbf_memory)

__all__ = [
    "CONFIGS", "BY_NAME", "Config", "KernelSpec", "dft", "green_cubes", "green_plates", "level_rule", "nudft",
    "radon2d", "radon3d",
    "ColumnID", "ProxyStrategy", "TensorButterfly", "column_id", "column_id_batch", "dense_rows", "derive_seed",
    "mode_product_blockdiag", "select_proxies", "select_proxies_count", "subtensor_at", "tbf_construct",
    "tbf_contract", "tbf_error_estimate", "tbf_load", "tbf_memory",
]
