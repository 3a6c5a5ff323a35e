"""B200-native inference from Deep-Compression-style models (arxiv 1711.00244).

Thin ctypes binding over libcdn.so (include/cdn.h).  Argument marshalling only:
every step of the hot path (Huffman decode, gap prefix sum, dequantize, sparse
multiply, bias, ReLU) runs in the library's CUDA kernels.  PyTorch is used only
for device memory, streams and process groups.  There is no CPU fallback: if
the library is missing or fails to load, importing the binding raises.
"""
from .binding import (CDN_SHARD_COLS, CDN_SHARD_ROWS, CDNError, LayerDesc, LayerStats, Model, abi_version,
                      col_block, compress_dense, debug_gemm_bf16,
                      kernel_launches, kernel_time, kernel_timer,
                      debug_host_walk, debug_host_walk_shard, lib_path, load_library, nccl_unique_id, plan_dp)

__all__ = ["CDN_SHARD_COLS", "CDN_SHARD_ROWS", "CDNError", "LayerDesc", "col_block", "LayerStats", "Model", "abi_version", "compress_dense",
           "debug_host_walk", "debug_host_walk_shard", "kernel_launches", "kernel_time", "kernel_timer", "lib_path", "load_library",
           "nccl_unique_id", "plan_dp"]
