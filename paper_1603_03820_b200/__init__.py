"""B200-native (sm_100a) ALS hot path of cuMF (arXiv 1603.03820) behind the reference
alskit API. Compute lives in libalskit_cuda.so (csrc/, C ABI in include/alskit_cuda.h);
`alskit` mirrors the reference's API, `session` keeps factors resident in HBM."""
from . import alskit  # noqa: F401  (loads libalskit_cuda.so; fails loudly if missing)

__all__ = ["alskit"]
