"""paper_2503_12964_b200 — B200-native shot-boundary clip splitting.

The data-parallel hot path of the NeMo Curator clipping pipeline of arXiv
2503.12964 (§2.1): per-frame colour histograms, adjacent-frame
colour-change cuts, and the embedding-similarity merge, as hand-written
sm_100a CUDA kernels behind a C ABI (include/clip_detect.h).
"""
from ._build import build  # noqa: F401
from .clipdetect import (Ctx, ClipError, default_params, load, run)  # noqa: F401
