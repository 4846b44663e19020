"""B200-native engine for the lookahead hot path of arXiv 2602.16760 (splitf).

The product is libsfg.so (CUDA for sm_100a + C++ host runtime) behind the C
ABI in include/sfg.h; this package is its thin Python mirror.
"""
from ._lib import SplitError, build, lib  # noqa: F401
from .engine import (  # noqa: F401
    EXACT, F16, F32, FAST, Batcher, CacheBank, DecodeResult, Engine, LookaheadConfig, ModelConfig, NGramPool,
    Router, ServerConfig, ServerEngine, SplitClient, SplitConfig, decode_lookahead, decode_lookahead_with_pool,
    decode_sequential, f16_bits_to_f32, f32_to_f16_bits, tp_unique_id)
