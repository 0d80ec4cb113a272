"""Seeded synthetic KV-cache inputs shared by the oracle side and the CUDA side of the tests.

This module holds NO arithmetic of the streaming method (no routing, no offsets, no packing). It
only answers "what 16-bit word does the writer put at LOGICAL coordinate (kv, layer, request,
head, position, d)", plus materialising a logical block as a numpy array (and, for the
FasterTransformer 6-D key structure, as that array's plain transpose).

Generators (SURVEY §8(c) C-3 and §8(d) "Synthetic inputs"):

* ``hash``  -- word = bits 48..63 of splitmix64(key(kv,l,r,h,s,d) XOR mix(seed)). Global
  coordinates make the content independent of partition and layout. Random 16-bit patterns include
  fp16 NaN/Inf/denormal encodings, so a path that routes words through float registers fails.
* ``uid``   -- word = row-major linear id of (kv,l,r,h,s,d) inside a global box; valid while the box
  has < 2**16 elements (the C1 toy: 2*2*2*4*40*16 = 20,480). Every word decodes back to its
  coordinate, so a transposed or shifted copy is visible.

The CUDA side implements the same counter-based generator in its own test kernel
(``dvt_fill`` in include/dv_testing.h); tests pin the two against each other bit-exactly.

Seeds: 20240304 + config number.
"""
from __future__ import annotations

import numpy as np

SENTINEL = 0xFFFF  # destination words outside the streamed region (an fp16 NaN) must stay this
POISON = 0xFFFE    # source words outside the written/streamed region; must never reach a destination

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_SEEDMUL = np.uint64(0xD1B54A32D192ED03)

# key(kv,l,r,h,s,d) bit fields: d[0:10) s[10:30) h[30:40) r[40:52) l[52:62) kv[62]
KEY_LIMITS = dict(d=1 << 10, s=1 << 20, h=1 << 10, r=1 << 12, l=1 << 10)


def config_seed(cfg: int) -> int:
    return 20240304 + cfg


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Steele/Lea/Flood splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def seed_mix(seed: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return np.uint64((int(seed) * int(_SEEDMUL)) & 0xFFFFFFFFFFFFFFFF)


def coord_key(kv, l, r, h, s, d) -> np.ndarray:
    u = lambda a: np.asarray(a, dtype=np.uint64)
    return ((u(kv) << np.uint64(62)) | (u(l) << np.uint64(52)) | (u(r) << np.uint64(40))
            | (u(h) << np.uint64(30)) | (u(s) << np.uint64(10)) | u(d))


def hash_words(kv, l, r, h, s, d, seed: int) -> np.ndarray:
    """16-bit word at logical coordinates (broadcasting arrays), generator ``hash``."""
    z = splitmix64(coord_key(kv, l, r, h, s, d) ^ seed_mix(seed))
    return (z >> np.uint64(48)).astype(np.uint16)


def uid_words(kv, l, r, h, s, d, box) -> np.ndarray:
    """Generator ``uid``: row-major id inside box=(L, R, H, S, D) (global extents, kv outermost)."""
    L, R, H, S, D = box
    if 2 * L * R * H * S * D > 1 << 16:
        raise ValueError("uid box too large for 16-bit ids")
    i = (((((np.asarray(kv) * L + l) * R + r) * H + h) * S + s) * D + d)
    return np.asarray(i, dtype=np.uint16)


def uid_decode(w: np.ndarray, box):
    """Inverse of uid_words: returns (kv, l, r, h, s, d) arrays."""
    L, R, H, S, D = box
    w = np.asarray(w, dtype=np.int64)
    d = w % D; w = w // D
    s = w % S; w = w // S
    h = w % H; w = w // H
    r = w % R; w = w // R
    l = w % L; kv = w // L
    return kv, l, r, h, s, d


def logical_block(kind: str, kv: int, layers, reqs, n_heads: int, positions, head_dim: int,
                  seed: int = 0, box=None, valid_pos=None, head_begin: int = 0) -> np.ndarray:
    """Logical array [nL][nR][H][nS][D] (uint16) of the writer's words.

    layers/reqs/positions are iterables of GLOBAL ids; heads are the global ids
    [head_begin, head_begin + n_heads) (a tensor-parallel shard). Positions outside ``valid_pos``
    (a half-open (lo, hi) pair, default: all) hold POISON -- the writer never produced them.
    """
    L = np.asarray(list(layers), dtype=np.int64)[:, None, None, None, None]
    R = np.asarray(list(reqs), dtype=np.int64)[None, :, None, None, None]
    Hh = np.arange(head_begin, head_begin + n_heads, dtype=np.int64)[None, None, :, None, None]
    P = np.asarray(list(positions), dtype=np.int64)[None, None, None, :, None]
    Dd = np.arange(head_dim, dtype=np.int64)[None, None, None, None, :]
    if kind == "hash":
        w = hash_words(kv, L, R, Hh, P, Dd, seed)
    elif kind == "uid":
        w = uid_words(kv, L, R, Hh, P, Dd, box)
    else:
        raise ValueError(kind)
    w = np.broadcast_to(w, (L.shape[0], R.shape[1], n_heads, P.shape[3], head_dim)).copy()
    if valid_pos is not None:
        lo, hi = valid_pos
        bad = (P[0, 0, 0, :, 0] < lo) | (P[0, 0, 0, :, 0] >= hi)
        w[:, :, :, bad, :] = POISON
    return w


def kv5d_cache(kind: str, layer_begin: int, n_layers: int, req_begin: int, n_reqs: int,
               n_heads: int, max_seq: int, head_dim: int, seed: int = 0, box=None,
               valid_pos=None, head_begin: int = 0):
    """(K, V) arrays in the [L][B][H][S][D] order the writer (FasterTransformer-style) fills.

    For this order the logical block IS the physical array, so no layout arithmetic is involved.
    """
    layers = range(layer_begin, layer_begin + n_layers)
    reqs = range(req_begin, req_begin + n_reqs)
    pos = range(max_seq)
    return tuple(logical_block(kind, kv, layers, reqs, n_heads, pos, head_dim, seed, box, valid_pos,
                               head_begin) for kv in (0, 1))


def as_ft6d_key(K: np.ndarray, elem_bytes: int = 2) -> np.ndarray:
    """Materialise a logical [L][B][H][S][D] key block in FasterTransformer's 6-D key structure
    [L][B][H][D/x][S][x], x = 16/elem_bytes (input STRUCTURE of NEXT-1; a plain transpose)."""
    x = 16 // elem_bytes
    nL, nR, H, S, D = K.shape
    return np.ascontiguousarray(K.reshape(nL, nR, H, S, D // x, x).transpose(0, 1, 2, 4, 3, 5))


def sentinel_cache(n_layers: int, n_reqs: int, n_heads: int, max_seq: int, head_dim: int):
    shape = (n_layers, n_reqs, n_heads, max_seq, head_dim)
    return (np.full(shape, SENTINEL, np.uint16), np.full(shape, SENTINEL, np.uint16))


def random_cache(n_layers: int, n_reqs: int, n_heads: int, max_seq: int, head_dim: int,
                 elem_bytes: int, seed: int):
    """(K, V) of random words of 1, 2, 4 or 8 bytes (e.g. fp8 / fp32 KV caches), seeded."""
    dt = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[elem_bytes]
    rng = np.random.default_rng(seed)
    shape = (n_layers, n_reqs, n_heads, max_seq, head_dim)
    return tuple(rng.integers(0, np.iinfo(dt).max, shape, dtype=dt, endpoint=True) for _ in range(2))
