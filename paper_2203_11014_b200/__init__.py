"""B200-native DHEN (arXiv 2203.11014) layer-stack training path.

The product is libdhen.so (C ABI: include/dhen.h, hand-written sm_100a CUDA);
`binding` is its thin ctypes binding."""
from .binding import (ATTN, BF16, CONV, DCN, DOT, FP32, LINEAR, MLP, Config, DHEN, DhenError, Module,  # noqa: F401
                      group_numel, load, nccl_id, sizes, validate)
