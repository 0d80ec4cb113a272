"""CPU ORACLE for DéjàVuLib KV-cache streaming -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this module. The CUDA product (``paper_2403_01876_b200``) never imports
it and shares no code with it; the two meet only through ``kvgen`` (seeded inputs, no method
arithmetic).

What it computes -- the plain definition of the streamed result:

    for kv in {K,V}, l in [l0,l1), r in [r0,r1), h in [0,H), s in [s0,s1), d in [0,D):
        i = stage of l in the source setup,   j = stage of l in the destination setup
        u = microbatch of r at the source,    w = microbatch of r at the destination
        T[j,w].kv[l - b_j][r - rho'_w][h][s][d] = S[i,u].kv[l - a_i][r - rho_u][h][s][d]
    every other word of every T is unchanged; no word of any S changes.

It is organised the way the paper's primitive levels are (Table 1):
``stream``  (stream_out/stream_in: find destinations, split/merge)  -> ``route``
``pack``/``unpack`` (scatter/gather: non-contiguous region <-> contiguous chunk)
``transfer`` (flush/fetch: copy one contiguous chunk)

Two modes of pack/unpack: ``brute`` (explicit nested loops, element by element; tiny shapes only)
and ``vector`` (numpy slicing). Tests check brute == vector.

Pins (tests/test_oracle_pins.py):
  region_bytes -- SPEC.md:35-43 worked example 37,748,736 B; SPEC.md:44-52 per-layer footprints.
  route        -- SPEC.md:376-378 split/merge examples; C3 7-piece list;
                  brute-force cell enumeration: every (layer, request) covered exactly once.
  pack/unpack  -- uid fill: every destination word decodes to the global coordinate it sits at;
                  sentinel outside the region unchanged; poison never copied.
  positions    -- Fig. 6 narrative: prompt of 4 fills [0,4), tokens fill 4 then 5.
  round trip   -- stream_out then stream_in restores the cache.
  swap         -- rotation examples; bytes = i*B*C.
  ring         -- x -> (x+1)%N, N-1 -> 0.
  recovery     -- Fig. 10 example, stage 2 of 4 fails.
Nothing here is "parity unpinned".

Readings of the paper where it is silent/ambiguous are SURVEY §8(c) C-4 Q1-Q18, restated in
DESIGN.md "Readings". Canonical wire order (Q3): [l][kv][r][h][s][d], d fastest.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

LAYOUT_KV5D = 0   # K and V both [L_s][B][H][S][D]                      (north_star; Q1)
LAYOUT_FT6D = 1   # K [L_s][B][H][D/x][S][x], x = 16/e ; V [L_s][B][H][S][D]  (PAPER.md:131 fn 5; NEXT-1)
# Regions are (l0, l1, r0, r1, s0, s1) -- all heads -- or (l0, l1, r0, r1, s0, s1, h0, h1) with
# GLOBAL head ids (tensor-parallel shards, NEXT-4); (h0, h1) == (0, 0) also means all heads.


class MappingError(ValueError):
    """Source/destination setups do not cover the region exactly once."""


class RangeError(ValueError):
    """A position range exceeds max_seq on one side ('naming the limit')."""


# --------------------------------------------------------------------------------------------
# Sizes (§2.1; "2 * hidden * element_bytes" per layer.token.request)
# --------------------------------------------------------------------------------------------
def region_bytes(layer_begin, layer_end, req_begin, req_end, pos_begin, pos_end,
                 n_heads, head_dim, elem_bytes) -> int:
    """Bytes of K and V in a region: 2 (K and V) * layers * requests * positions * H * D * e.

    SPEC.md:38 "2 * L * hidden * element_bytes * batch * seq" with hidden = H * D.
    """
    nL = layer_end - layer_begin
    nR = req_end - req_begin
    n = pos_end - pos_begin
    if nL < 0 or nR < 0 or n < 0:
        raise ValueError("negative extent")
    return 2 * nL * nR * n * n_heads * head_dim * elem_bytes


# --------------------------------------------------------------------------------------------
# Setups and routing (stream_out / stream_in level: PAPER.md:169-172 Table 1, :266 §4.2.1)
# --------------------------------------------------------------------------------------------
@dataclass
class Setup:
    """A pipeline configuration: layer partition over stages (PP), request split into
    microbatches and, optionally, head split over tensor-parallel ranks
    inside a stage. Bounds are global ids, half-open, strictly
    increasing. head_bounds None = no head split (every block holds all heads)."""
    layer_bounds: List[int]
    req_bounds: List[int]
    max_seq: int
    head_bounds: Optional[List[int]] = None

    @property
    def n_stages(self):
        return len(self.layer_bounds) - 1

    @property
    def n_micro(self):
        return len(self.req_bounds) - 1

    @property
    def n_tp(self):
        return 1 if self.head_bounds is None else len(self.head_bounds) - 1

    def flat(self, stage, micro, tp=0):
        """Flat block index (stage*n_micro + micro)*n_tp + tp."""
        return (stage * self.n_micro + micro) * self.n_tp + tp


def even_layer_bounds(n_layers: int, n_stages: int, layer_begin: int = 0) -> List[int]:
    """Reading Q6 (PAPER.md:196 assumes T_n divides L): the first L mod P stages get ceil(L/P)."""
    q, rem = divmod(n_layers, n_stages)
    b = [layer_begin]
    for st in range(n_stages):
        b.append(b[-1] + q + (1 if st < rem else 0))
    return b


@dataclass
class Piece:
    src_stage: int
    src_micro: int
    dst_stage: int
    dst_micro: int
    layer_begin: int
    layer_end: int
    req_begin: int
    req_end: int
    pos_begin: int
    pos_end: int
    bytes: int = 0
    src_wire_off: int = 0
    dst_wire_off: int = 0
    src_tp: int = 0
    dst_tp: int = 0
    head_begin: int = 0          # [0,0): all heads (no setup splits heads)
    head_end: int = 0

    def region(self):
        r = (self.layer_begin, self.layer_end, self.req_begin, self.req_end, self.pos_begin, self.pos_end)
        if self.head_end > self.head_begin:
            r = r + (self.head_begin, self.head_end)
        return r


def _check_setup(s: Setup, name: str):
    bounds = [s.layer_bounds, s.req_bounds] + ([s.head_bounds] if s.head_bounds is not None else [])
    for b in bounds:
        if len(b) < 2 or b[0] < 0 or any(b[k + 1] <= b[k] for k in range(len(b) - 1)):
            raise ValueError(f"{name}: bounds must be non-negative, strictly increasing, >= 1 block")
    if s.max_seq < 1:
        raise ValueError(f"{name}: max_seq must be >= 1")


def split_region(region):
    """(l0,l1,r0,r1,s0,s1[,h0,h1]) -> (l0,l1,r0,r1,s0,s1, heads or None for 'all heads')."""
    if len(region) == 6:
        return (*region, None)
    l0, l1, r0, r1, s0, s1, h0, h1 = region
    return l0, l1, r0, r1, s0, s1, (None if (h0, h1) == (0, 0) else (h0, h1))


def route(src: Setup, dst: Setup, region, n_heads: int, head_dim: int, elem_bytes: int) -> List[Piece]:
    """Pieces = non-empty intersections  region x src block (i,u,t) x dst block (j,w,v).

    Plain loops in the order (i, u, t, j, w, v), i.e. by flat source block then flat destination
    block. ``bytes`` is the piece's wire size (heads = the piece's head range, or ``n_heads`` when
    no setup splits heads); ``src_wire_off`` is the offset of the piece among the pieces leaving its
    source block, ``dst_wire_off`` among the pieces entering its destination block, cumulative in
    that loop order.

    Errors, checked in this order: ValueError for a malformed setup or region, or when exactly one
    setup splits heads; MappingError unless both setups hold the region's layers, requests and
    heads; RangeError if pos_end exceeds max_seq on either side. An
    empty region (any extent 0) routes to no pieces.
    """
    l0, l1, r0, r1, s0, s1, heads = split_region(region)
    _check_setup(src, "source setup")
    _check_setup(dst, "destination setup")
    if (src.head_bounds is None) != (dst.head_bounds is None):
        raise ValueError("both setups or neither must split heads")
    if not (l0 <= l1 and r0 <= r1 and 0 <= s0 <= s1) or (heads is not None and not 0 <= heads[0] <= heads[1]):
        raise ValueError("malformed region")
    tp = src.head_bounds is not None
    if tp and heads is None:
        heads = (src.head_bounds[0], src.head_bounds[-1])
    if l0 == l1 or r0 == r1 or s0 == s1 or (heads is not None and heads[0] == heads[1]):
        return []                      # empty region: nothing to move (still a valid call)
    for nm, s in (("source", src), ("destination", dst)):
        if l0 < s.layer_bounds[0] or l1 > s.layer_bounds[-1]:
            raise MappingError(f"{nm} setup does not hold layers [{l0},{l1})")
        if r0 < s.req_bounds[0] or r1 > s.req_bounds[-1]:
            raise MappingError(f"{nm} setup does not hold requests [{r0},{r1})")
        if tp and (heads[0] < s.head_bounds[0] or heads[1] > s.head_bounds[-1]):
            raise MappingError(f"{nm} setup does not hold heads [{heads[0]},{heads[1]})")
    for nm, s in (("source", src), ("destination", dst)):
        if s1 > s.max_seq:
            raise RangeError(f"pos_end {s1} exceeds {nm} max_seq {s.max_seq}")
    sh = src.head_bounds if tp else [0, 0]
    dh = dst.head_bounds if tp else [0, 0]
    pieces: List[Piece] = []
    for i in range(src.n_stages):
        for u in range(src.n_micro):
            for t in range(src.n_tp):
                for j in range(dst.n_stages):
                    for w in range(dst.n_micro):
                        for v in range(dst.n_tp):
                            a = max(l0, src.layer_bounds[i], dst.layer_bounds[j])
                            b = min(l1, src.layer_bounds[i + 1], dst.layer_bounds[j + 1])
                            c = max(r0, src.req_bounds[u], dst.req_bounds[w])
                            d = min(r1, src.req_bounds[u + 1], dst.req_bounds[w + 1])
                            if tp:
                                e = max(heads[0], sh[t], dh[v])
                                f = min(heads[1], sh[t + 1], dh[v + 1])
                            else:
                                e, f = (heads if heads is not None else (0, 0))
                            if a < b and c < d and (not tp or e < f):
                                p = Piece(i, u, j, w, a, b, c, d, s0, s1, src_tp=t, dst_tp=v,
                                          head_begin=e, head_end=f)
                                nh = (f - e) if (tp or heads is not None) else n_heads
                                p.bytes = region_bytes(a, b, c, d, s0, s1, nh, head_dim, elem_bytes)
                                pieces.append(p)
    src_acc: Dict[Tuple[int, int, int], int] = {}
    dst_acc: Dict[Tuple[int, int, int], int] = {}
    for p in pieces:
        ks, kd = (p.src_stage, p.src_micro, p.src_tp), (p.dst_stage, p.dst_micro, p.dst_tp)
        p.src_wire_off = src_acc.get(ks, 0)
        src_acc[ks] = p.src_wire_off + p.bytes
        p.dst_wire_off = dst_acc.get(kd, 0)
        dst_acc[kd] = p.dst_wire_off + p.bytes
    return pieces


# --------------------------------------------------------------------------------------------
# Caches (PAPER.md:47, 119 preallocated to max_seq; :131 fn 5 dimensionality)
# --------------------------------------------------------------------------------------------
@dataclass
class Cache:
    """One worker's K and V cache for layers [layer_begin, +n_layers), requests
    [req_begin, +n_reqs) and heads [head_begin, +n_heads) (a tensor-parallel shard), preallocated
    to max_seq."""
    K: np.ndarray
    V: np.ndarray
    layer_begin: int
    req_begin: int
    n_heads: int
    max_seq: int
    head_dim: int
    layout: int = LAYOUT_KV5D
    head_begin: int = 0

    @property
    def n_layers(self):
        return self.K.shape[0]

    @property
    def n_reqs(self):
        return self.K.shape[1]

    @property
    def elem_bytes(self):
        return self.K.dtype.itemsize

    def copy(self):
        return Cache(self.K.copy(), self.V.copy(), self.layer_begin, self.req_begin,
                     self.n_heads, self.max_seq, self.head_dim, self.layout, self.head_begin)

    # --- element addressing: the ONE place where the physical layout is spelled out ---------
    def word_index(self, kv, l, r, h, s, d):
        """Index tuple into self.K / self.V for GLOBAL layer l, request r and head h."""
        lp, rp, hp = l - self.layer_begin, r - self.req_begin, h - self.head_begin
        if self.layout == LAYOUT_FT6D and kv == 0:
            x = 16 // self.elem_bytes
            return (lp, rp, hp, d // x, s, d % x)
        return (lp, rp, hp, s, d)

    def arr(self, kv):
        return self.K if kv == 0 else self.V

    def heads_of(self, heads):
        return (self.head_begin, self.head_begin + self.n_heads) if heads is None else heads

    def holds(self, l0, l1, r0, r1, s1, heads=None):
        h0, h1 = self.heads_of(heads)
        return (self.layer_begin <= l0 and l1 <= self.layer_begin + self.n_layers
                and self.req_begin <= r0 and r1 <= self.req_begin + self.n_reqs
                and self.head_begin <= h0 and h1 <= self.head_begin + self.n_heads
                and s1 <= self.max_seq)

    def logical(self, kv, l0, l1, r0, r1, s0, s1, heads=None):
        """Logical view [l][r][h][s][d] of a region (copy)."""
        a = self.arr(kv)
        h0, h1 = self.heads_of(heads)
        lp = slice(l0 - self.layer_begin, l1 - self.layer_begin)
        rp = slice(r0 - self.req_begin, r1 - self.req_begin)
        hp = slice(h0 - self.head_begin, h1 - self.head_begin)
        if self.layout == LAYOUT_FT6D and kv == 0:
            # [l][r][h][D/x][s][x] -> [l][r][h][s][D/x][x] -> [l][r][h][s][D]
            blk = a[lp, rp, hp, :, s0:s1, :]
            blk = blk.transpose(0, 1, 2, 4, 3, 5)
            return blk.reshape(blk.shape[0], blk.shape[1], blk.shape[2], blk.shape[3], -1).copy()
        return a[lp, rp, hp, s0:s1, :].copy()

    def set_logical(self, kv, l0, l1, r0, r1, s0, s1, blk, heads=None):
        a = self.arr(kv)
        h0, h1 = self.heads_of(heads)
        lp = slice(l0 - self.layer_begin, l1 - self.layer_begin)
        rp = slice(r0 - self.req_begin, r1 - self.req_begin)
        hp = slice(h0 - self.head_begin, h1 - self.head_begin)
        if self.layout == LAYOUT_FT6D and kv == 0:
            x = 16 // self.elem_bytes
            b6 = blk.reshape(blk.shape[0], blk.shape[1], blk.shape[2], blk.shape[3], -1, x)
            a[lp, rp, hp, :, s0:s1, :] = b6.transpose(0, 1, 2, 4, 3, 5)
        else:
            a[lp, rp, hp, s0:s1, :] = blk


def make_cache(K, V, layer_begin, req_begin, n_heads, max_seq, head_dim, layout=LAYOUT_KV5D, head_begin=0):
    return Cache(np.asarray(K), np.asarray(V), layer_begin, req_begin, n_heads, max_seq,
                 head_dim, layout, head_begin)


def _check_holds(c: Cache, region, what):
    l0, l1, r0, r1, s0, s1, heads = split_region(region)
    if s1 > c.max_seq:
        raise RangeError(f"pos_end {s1} exceeds {what} max_seq {c.max_seq}")
    if not c.holds(l0, l1, r0, r1, s1, heads):
        raise MappingError(f"{what} cache does not hold the region")


# --------------------------------------------------------------------------------------------
# scatter / gather level (Table 1; Opt (1) buffered copies PAPER.md:121)
# --------------------------------------------------------------------------------------------
def wire_index(region, n_heads, head_dim, l, kv, r, h, s, d) -> int:
    """Word index of (l,kv,r,h,s,d) in the canonical wire chunk of ``region`` (reading Q3):
    dense [l-l0][kv][r-r0][h-h0][s-s0][d]; with a 6-tuple region the heads are [0, n_heads)."""
    l0, l1, r0, r1, s0, s1, heads = split_region(region)
    h0, h1 = heads if heads is not None else (0, n_heads)
    nR, n, nH = r1 - r0, s1 - s0, h1 - h0
    return (((((l - l0) * 2 + kv) * nR + (r - r0)) * nH + (h - h0)) * n + (s - s0)) * head_dim + d


def pack(src: Cache, region, mode: str = "vector") -> np.ndarray:
    """Non-contiguous region of ``src`` -> one contiguous wire chunk (the paper's ``scatter`` with
    Opt (1): "aggregate all updates in a temporary buffer")."""
    _check_holds(src, region, "source")
    l0, l1, r0, r1, s0, s1, heads = split_region(region)
    h0, h1 = src.heads_of(heads)
    D = src.head_dim
    reg = (l0, l1, r0, r1, s0, s1, h0, h1)
    nwords = region_bytes(l0, l1, r0, r1, s0, s1, h1 - h0, D, src.elem_bytes) // src.elem_bytes
    if mode == "brute":
        wire = np.empty(nwords, src.K.dtype)
        for l in range(l0, l1):
            for kv in (0, 1):
                for r in range(r0, r1):
                    for h in range(h0, h1):
                        for s in range(s0, s1):
                            for d in range(D):
                                wire[wire_index(reg, 0, D, l, kv, r, h, s, d)] = \
                                    src.arr(kv)[src.word_index(kv, l, r, h, s, d)]
        return wire
    blocks = [src.logical(kv, l0, l1, r0, r1, s0, s1, (h0, h1)) for kv in (0, 1)]  # [l][r][h][s][d]
    wire = np.stack(blocks, axis=1)                                                # [l][kv][r][h][s][d]
    return np.ascontiguousarray(wire).reshape(-1)


def unpack(dst: Cache, region, wire: np.ndarray, mode: str = "vector") -> None:
    """Contiguous wire chunk -> region of ``dst`` (the paper's ``gather``). The
    destination may have another max_seq, layer, request or head offset."""
    _check_holds(dst, region, "destination")
    l0, l1, r0, r1, s0, s1, heads = split_region(region)
    h0, h1 = dst.heads_of(heads)
    D = dst.head_dim
    reg = (l0, l1, r0, r1, s0, s1, h0, h1)
    nwords = region_bytes(l0, l1, r0, r1, s0, s1, h1 - h0, D, dst.elem_bytes) // dst.elem_bytes
    if wire.size != nwords:
        raise ValueError(f"wire has {wire.size} words, region needs {nwords}")
    if mode == "brute":
        for l in range(l0, l1):
            for kv in (0, 1):
                for r in range(r0, r1):
                    for h in range(h0, h1):
                        for s in range(s0, s1):
                            for d in range(D):
                                dst.arr(kv)[dst.word_index(kv, l, r, h, s, d)] = \
                                    wire[wire_index(reg, 0, D, l, kv, r, h, s, d)]
        return
    w = wire.reshape(l1 - l0, 2, r1 - r0, h1 - h0, s1 - s0, D)
    for kv in (0, 1):
        dst.set_logical(kv, l0, l1, r0, r1, s0, s1, w[:, kv], (h0, h1))


def shifted(region, k):
    """`region` moved k positions later."""
    return tuple(region[:4]) + (region[4] + k, region[5] + k) + tuple(region[6:])


def unpack_chunks(dst: Cache, first, log: np.ndarray, n_chunks: int, pos_step: int,
                  mode: str = "vector") -> None:
    """A log of chunks (host log form of a swap arena, reading of PAPER.md:270/572): chunk k is the
    wire of `first` shifted by k*pos_step positions, stored back to back. Unpack them in order."""
    e = dst.elem_bytes
    l0, l1, r0, r1, s0, s1, heads = split_region(first)
    h0, h1 = dst.heads_of(heads)
    w = region_bytes(l0, l1, r0, r1, s0, s1, h1 - h0, dst.head_dim, e) // e
    for k in range(n_chunks):
        unpack(dst, shifted(first, k * pos_step), log[k * w:(k + 1) * w], mode)


def transfer(wire: np.ndarray) -> np.ndarray:
    """flush / fetch: copy one contiguous chunk. On the CPU: a byte copy."""
    return np.frombuffer(bytes(wire.tobytes()), dtype=wire.dtype).copy()


def remap(src: Cache, dst: Cache, region, mode: str = "vector") -> None:
    """Direct layout-to-layout copy of a region (pack -> transfer -> unpack composed). A 6-tuple
    region means the source cache's heads."""
    l0, l1, r0, r1, s0, s1, heads = split_region(region)
    reg = (l0, l1, r0, r1, s0, s1) + src.heads_of(heads)
    unpack(dst, reg, transfer(pack(src, reg, mode)), mode)


# --------------------------------------------------------------------------------------------
# stream_out / stream_in level (Table 1; §4.2.1 split/merge PAPER.md:266)
# --------------------------------------------------------------------------------------------
def _bkey(setup: Setup, stage, micro, tp):
    """Block key: (stage, micro) without tensor parallelism, (stage, micro, tp) with it."""
    return (stage, micro) if setup.head_bounds is None else (stage, micro, tp)


def stream_out(src_caches: Dict[tuple, Cache], src: Setup, dst: Setup, region,
               mode: str = "vector") -> Dict[tuple, np.ndarray]:
    """Every source block packs each of its pieces and flushes it into the destination block's
    inbox at the piece's ``dst_wire_off``. Returns the inboxes {dst block key: wire words}."""
    any_c = next(iter(src_caches.values()))
    H, D, e = any_c.n_heads, any_c.head_dim, any_c.elem_bytes
    pieces = route(src, dst, region, H, D, e)
    inbox_words: Dict[tuple, int] = {}
    for p in pieces:
        k = _bkey(dst, p.dst_stage, p.dst_micro, p.dst_tp)
        inbox_words[k] = max(inbox_words.get(k, 0), (p.dst_wire_off + p.bytes) // e)
    inboxes = {k: np.zeros(n, any_c.K.dtype) for k, n in inbox_words.items()}
    for p in pieces:
        sc = src_caches[_bkey(src, p.src_stage, p.src_micro, p.src_tp)]
        wire = transfer(pack(sc, p.region(), mode))
        o = p.dst_wire_off // e
        inboxes[_bkey(dst, p.dst_stage, p.dst_micro, p.dst_tp)][o:o + wire.size] = wire
    return inboxes


def stream_in(dst_caches: Dict[tuple, Cache], src: Setup, dst: Setup, region,
              inboxes: Dict[tuple, np.ndarray], mode: str = "vector") -> None:
    """Every destination block unpacks each piece addressed to it from its inbox."""
    any_c = next(iter(dst_caches.values()))
    H, D, e = any_c.n_heads, any_c.head_dim, any_c.elem_bytes
    for p in route(src, dst, region, H, D, e):
        k = _bkey(dst, p.dst_stage, p.dst_micro, p.dst_tp)
        o = p.dst_wire_off // e
        unpack(dst_caches[k], p.region(), inboxes[k][o:o + p.bytes // e], mode)


def stream(src_caches, src: Setup, dst_caches, dst: Setup, region, mode: str = "vector"):
    """stream_out followed by stream_in; mutates dst_caches in place and returns them."""
    stream_in(dst_caches, src, dst, region, stream_out(src_caches, src, dst, region, mode), mode)
    return dst_caches


# --------------------------------------------------------------------------------------------
# Scenario rules (§4.2.2 swapping, §4.2.3 replication / recovery)
# --------------------------------------------------------------------------------------------
def token_position(prompt_len: int, step: int) -> int:
    """Reading Q4 (Fig. 6): the prompt fills [0,p); token step t>=1 writes p+t-1."""
    if step < 1:
        raise ValueError("token steps start at 1")
    return prompt_len + step - 1


def swap_rotation(x: int, n: int) -> Tuple[int, int]:
    """"when microbatch x is processed, microbatch (x+1)%N is swapped in, and
    microbatch (x-1)%N is swapped out". Returns (swap_in, swap_out)."""
    if n < 2 or not 0 <= x < n:
        raise ValueError("need N >= 2 and 0 <= x < N")
    return (x + 1) % n, (x - 1) % n


def swap_budget(depth: int, per_micro_bytes: int) -> Tuple[int, int]:
    """PAPER.md:270 "D*M GB in CPU memory, and 2*M GB in GPU memory" + fn 6 (:274) "or M GB in GPU
    memory if D == 2". Returns (host_bytes, device_bytes)."""
    return depth * per_micro_bytes, (per_micro_bytes if depth == 2 else 2 * per_micro_bytes)


def swap_in_bytes(i: int, batch: int, c_bytes: int) -> int:
    """PAPER.md:572 transf_i = i*B*C_i/pciebw: the swap-in moves the whole prefix of length i."""
    return i * batch * c_bytes


def ring_successor(x: int, n: int) -> int:
    """worker x streams its KV cache to worker (x+1)%N."""
    return (x + 1) % n


def recovery_copies(x: int, n: int) -> List[Tuple[int, int, str]]:
    """(1) (x+1)%N sends the replica it hosts to x; (2) (x-1)%N sends its own cache to
    x (repopulating the replica x hosted). Returns [(from, to, what)]."""
    return [((x + 1) % n, x, "replica_of_x"), ((x - 1) % n, x, "own_cache_of_prev")]
