"""Test helpers for NV12 (reading O0): an image holding every (Y, U, V)
combination and the oracle's bin of every (Y, U, V).  Uses only oracle/."""
import numpy as np

import oracle

H_ALL = W_ALL = 4096  # 2048 x 2048 chroma blocks = 2^22 (U, V, Y-quad) triples


def all_yuv_image():
    """NV12 frame [H*3/2, W] in which block b = (by, bx) has U = b & 255,
    V = (b >> 8) & 255 and luma 4*(b >> 16) + k for its pixels k = 0..3
    (row-major within the 2x2 block): every (Y, U, V) appears exactly once."""
    H, W = H_ALL, W_ALL
    b = np.arange((H // 2) * (W // 2), dtype=np.int64)
    U, V, yb = b & 255, (b >> 8) & 255, b >> 16
    img = np.empty((H * 3 // 2, W), np.uint8)
    by, bx = np.divmod(b, W // 2)
    Ys = [4 * yb + k for k in range(4)]
    img[2 * by, 2 * bx], img[2 * by, 2 * bx + 1] = Ys[0], Ys[1]
    img[2 * by + 1, 2 * bx], img[2 * by + 1, 2 * bx + 1] = Ys[2], Ys[3]
    uv = img[H:].reshape(H // 2, W // 2, 2)
    uv[by, bx, 0], uv[by, bx, 1] = U, V
    return img, (by, bx, U, V, Ys)


def yuv_rgb_table():
    """oracle O0 RGB of every (Y, U, V): int64 [(Y << 16) | (U << 8) | V] -> (r << 16) | (g << 8) | b."""
    img, (by, bx, U, V, Ys) = all_yuv_image()
    rgb = oracle.nv12_to_rgb(img).astype(np.int64)
    out = np.empty(1 << 24, np.int64)
    for k, (dy, dx) in enumerate([(0, 0), (0, 1), (1, 0), (1, 1)]):
        px = rgb[2 * by + dy, 2 * bx + dx]
        out[(Ys[k] << 16) | (U << 8) | V] = (px[:, 0] << 16) | (px[:, 1] << 8) | px[:, 2]
    return out


def yuv_bins(p=oracle.Params()):
    """oracle O0 then O1: bin of every (Y, U, V), u8 [(Y << 16) | (U << 8) | V]."""
    return oracle.bin_table(p)[yuv_rgb_table()]


def random_nv12(rng, n, H, W, structured=False):
    """n random NV12 frames u8 [n, H*3/2, W]; structured = smooth blocks (few
    distinct colours, like decoded video) instead of uniform noise."""
    if not structured:
        return rng.integers(0, 256, size=(n, H * 3 // 2, W), dtype=np.uint8)
    out = np.empty((n, H * 3 // 2, W), np.uint8)
    for i in range(n):
        pal = rng.integers(0, 256, size=(8, 3))
        cells = rng.integers(0, 8, size=(H // 16 + 1, W // 16 + 1))
        yy, xx = np.mgrid[0:H, 0:W]
        k = cells[yy // 16, xx // 16]
        out[i, :H] = np.clip(pal[k, 0] + rng.integers(-4, 5, size=(H, W)), 0, 255)
        kb = cells[(2 * yy[:H // 2, :W // 2]) // 16, (2 * xx[:H // 2, :W // 2]) // 16]
        uv = out[i, H:].reshape(H // 2, W // 2, 2)
        uv[..., 0] = pal[kb, 1]
        uv[..., 1] = pal[kb, 2]
    return out
