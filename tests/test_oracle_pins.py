"""Pins for the CPU oracle against what the paper and the mathematics fix (no GPU).

Every check here compares the oracle with something other than itself: a number printed in
SPEC.md / the paper (tests/golden/*.json, each with its citation), brute-force enumeration on tiny
shapes, the uid fill (each word encodes its own coordinate), or kvgen's direct definition of what
the writer put at a logical coordinate.
"""
import itertools
import random

import numpy as np
import pytest

import kvgen
import oracle
from oracle import scenarios
from oracle.kvstream import (LAYOUT_FT6D, LAYOUT_KV5D, Cache, MappingError, RangeError, Setup,
                             even_layer_bounds, pack, region_bytes, remap, route, stream,
                             stream_in, stream_out, unpack)


# ---------------------------------------------------------------------------------------------
# byte formulas
# ---------------------------------------------------------------------------------------------
def test_region_bytes_spec_examples(golden):
    g = golden("spec_kv_bytes.json")
    for ex in g["kv_cache_bytes"]:
        H, D = 12, 64  # hidden 768 = H * D
        assert H * D == ex["hidden"]
        got = region_bytes(0, ex["layers"], 0, ex["batch"], 0, ex["seq"], H, D, ex["elem_bytes"])
        assert got == ex["bytes"], ex["cite"]
    for ex in g["footprints"]:
        H, D = 12, 64
        per = region_bytes(0, 1, 0, ex["batch"], 0, 1, H, D, ex["elem_bytes"])
        if "token_step_per_layer" in ex:
            assert per == ex["token_step_per_layer"]
        assert region_bytes(0, 1, 0, ex["batch"], 0, ex["prompt"], H, D, 2) == ex["prompt_per_layer"]


def test_pack_size_matches_spec_worked_example(golden):
    """The packed wire of a whole L=12, hidden=768, b=1, s=1024 fp16 cache is exactly the
    37,748,736 B of SPEC.md:42 -- pins pack's output size against the paper-derived formula."""
    ex = golden("spec_kv_bytes.json")["kv_cache_bytes"][0]
    H, D = 12, 64
    K, V = kvgen.kv5d_cache("hash", 0, 12, 0, 1, H, 1024, D, seed=1)
    c = Cache(K, V, 0, 0, H, 1024, D)
    wire = pack(c, (0, 12, 0, 1, 0, 1024))
    assert wire.nbytes == ex["bytes"]
    # linearity in batch
    K2, V2 = kvgen.kv5d_cache("hash", 0, 1, 0, 2, H, 1024, D, seed=1)
    c2 = Cache(K2, V2, 0, 0, H, 1024, D)
    assert pack(c2, (0, 1, 0, 2, 0, 1024)).nbytes * 12 == golden("spec_kv_bytes.json")["kv_cache_bytes"][1]["bytes"]


# ---------------------------------------------------------------------------------------------
# route (Table 1 stream_out/stream_in)
# ---------------------------------------------------------------------------------------------
def _pieces_as(pieces, fields):
    return [[getattr(p, f) for f in fields] for p in pieces]


def test_route_spec_depth_split(golden):
    g = golden("spec_route_examples.json")["depth_2_to_4_L24"]
    src = Setup(g["src_layer_bounds"], [0, 4], 64)
    dst = Setup(g["dst_layer_bounds"], [0, 4], 64)
    ps = route(src, dst, (0, 24, 0, 4, 0, 10), 2, 8, 2)
    assert _pieces_as(ps, ["src_stage", "dst_stage", "layer_begin", "layer_end"]) == g["pieces"]
    # merge is the inverse direction: 4 -> 2 gives the same 4 pieces with stages swapped
    ps_inv = route(dst, src, (0, 24, 0, 4, 0, 10), 2, 8, 2)
    assert sorted(_pieces_as(ps_inv, ["dst_stage", "src_stage", "layer_begin", "layer_end"])) == g["pieces"]


def test_route_spec_identity(golden):
    g = golden("spec_route_examples.json")["identity"]
    s = Setup(g["layer_bounds"], g["req_bounds"], 32)
    ps = route(s, s, (0, 30, 0, 8, 0, 32), 2, 8, 2)
    assert len(ps) == len(g["layer_bounds"]) - 1
    for k, p in enumerate(ps):
        assert (p.src_stage, p.dst_stage) == (k, k)
        assert (p.layer_begin, p.layer_end) == (g["layer_bounds"][k], g["layer_bounds"][k + 1])
        assert p.src_wire_off == 0 and p.dst_wire_off == 0


def test_route_spec_batch_split(golden):
    g = golden("spec_route_examples.json")["batch_16_to_8"]
    src = Setup([0, 4], g["src_req_bounds"], 16)
    dst = Setup([0, 4], g["dst_req_bounds"], 16)
    ps = route(src, dst, (0, 4, 0, 16, 0, 16), 2, 8, 2)
    assert _pieces_as(ps, ["src_micro", "dst_micro", "req_begin", "req_end"]) == g["pieces"]
    # the source slab is split: second half starts where the first half's bytes end
    assert ps[1].src_wire_off == ps[0].bytes
    assert ps[0].dst_wire_off == 0 and ps[1].dst_wire_off == 0


def test_route_c3_seven_pieces(golden):
    g = golden("c3_pieces.json")
    src = Setup(g["prompt_layer_bounds"], [0, 8], 1024)
    dst = Setup(g["token_layer_bounds"], [0, 8], 2048)
    ps = route(src, dst, (0, 64, 0, 8, 0, 1000), 72, 128, 2)
    assert _pieces_as(ps, ["src_stage", "dst_stage", "layer_begin", "layer_end"]) == g["pieces"]
    src16 = Setup(g["prompt_layer_bounds"], [0, 16], 1024)
    dst2x8 = Setup(g["token_layer_bounds"], [0, 8, 16], 2048)
    assert len(route(src16, dst2x8, (0, 64, 0, 16, 0, 1000), 72, 128, 2)) == \
        g["batch_split_16_to_2x8_piece_count"]
    # token stage 1 receives [13,16) from P0 then [16,30) from P1: inbox offsets follow piece order
    t1 = [p for p in ps if p.dst_stage == 1]
    C = 2 * 72 * 128 * 2 * 8 * 1000  # bytes per layer of the piece
    assert [(p.dst_wire_off, p.bytes) for p in t1] == [(0, 3 * C), (3 * C, 14 * C)]


def _random_bounds(rng, lo, hi, k):
    cuts = sorted(rng.sample(range(lo + 1, hi), k - 1)) if k > 1 else []
    return [lo] + cuts + [hi]


@pytest.mark.parametrize("seed", range(40))
def test_route_brute_force_coverage(seed):
    """Brute force: every (layer, request) cell of the region is covered by exactly one piece, that
    piece's source/destination blocks really hold the cell, byte counts add up, and the wire
    offsets of each destination (and source) block tile [0, total) without gaps or overlaps
    ("no piece lost, none duplicated")."""
    rng = random.Random(seed)
    L, R = rng.randint(1, 12), rng.randint(1, 9)
    src = Setup(_random_bounds(rng, 0, L, rng.randint(1, min(L, 4))),
                _random_bounds(rng, 0, R, rng.randint(1, min(R, 3))), 64)
    dst = Setup(_random_bounds(rng, 0, L, rng.randint(1, min(L, 4))),
                _random_bounds(rng, 0, R, rng.randint(1, min(R, 3))), 48)
    l0 = rng.randint(0, L - 1); l1 = rng.randint(l0 + 1, L)
    r0 = rng.randint(0, R - 1); r1 = rng.randint(r0 + 1, R)
    s0 = rng.randint(0, 20); s1 = rng.randint(s0 + 1, 48)
    H, D, e = 3, 8, 2
    ps = route(src, dst, (l0, l1, r0, r1, s0, s1), H, D, e)
    for l in range(L):
        for r in range(R):
            cov = [p for p in ps if p.layer_begin <= l < p.layer_end and p.req_begin <= r < p.req_end]
            inside = l0 <= l < l1 and r0 <= r < r1
            assert len(cov) == (1 if inside else 0)
            if cov:
                p = cov[0]
                assert src.layer_bounds[p.src_stage] <= l < src.layer_bounds[p.src_stage + 1]
                assert dst.layer_bounds[p.dst_stage] <= l < dst.layer_bounds[p.dst_stage + 1]
                assert src.req_bounds[p.src_micro] <= r < src.req_bounds[p.src_micro + 1]
                assert dst.req_bounds[p.dst_micro] <= r < dst.req_bounds[p.dst_micro + 1]
    for p in ps:
        assert p.bytes == 2 * (p.layer_end - p.layer_begin) * (p.req_end - p.req_begin) * (s1 - s0) * H * D * e
    assert sum(p.bytes for p in ps) == 2 * (l1 - l0) * (r1 - r0) * (s1 - s0) * H * D * e
    for key in (("dst_stage", "dst_micro", "dst_wire_off"), ("src_stage", "src_micro", "src_wire_off")):
        blocks = {}
        for p in ps:
            blocks.setdefault((getattr(p, key[0]), getattr(p, key[1])), []).append((getattr(p, key[2]), p.bytes))
        for spans in blocks.values():
            spans.sort()
            pos = 0
            for off, nb in spans:
                assert off == pos
                pos += nb


def test_route_errors():
    s = Setup([0, 4, 8], [0, 4], 32)
    with pytest.raises(MappingError):          # destination lacks layers 8..9
        route(Setup([0, 10], [0, 4], 32), s, (0, 10, 0, 4, 0, 8), 2, 8, 2)
    with pytest.raises(MappingError):          # requests not held
        route(s, s, (0, 8, 0, 5, 0, 8), 2, 8, 2)
    with pytest.raises(RangeError, match="max_seq 16"):  # names the limit
        route(s, Setup([0, 8], [0, 4], 16), (0, 8, 0, 4, 0, 17), 2, 8, 2)
    with pytest.raises(ValueError):
        route(Setup([0, 4, 4], [0, 4], 8), s, (0, 4, 0, 4, 0, 2), 2, 8, 2)
    assert route(s, s, (0, 8, 0, 4, 5, 5), 2, 8, 2) == []    # empty position range


def test_even_layer_bounds_reading_q6():
    assert even_layer_bounds(70, 8) == [0, 9, 18, 27, 36, 45, 54, 62, 70]   # BLOOM 70 over 8
    assert even_layer_bounds(64, 4) == [0, 16, 32, 48, 64]


# ---------------------------------------------------------------------------------------------
# pack / unpack (Table 1 scatter/gather; Opt (1))
# ---------------------------------------------------------------------------------------------
def _uid_cache(layer_begin, nL, req_begin, nR, H, S, D, box, valid=None, layout=LAYOUT_KV5D):
    K, V = kvgen.kv5d_cache("uid", layer_begin, nL, req_begin, nR, H, S, D, box=box, valid_pos=valid)
    c = Cache(K, V, layer_begin, req_begin, H, S, D)
    if layout == LAYOUT_FT6D:
        c = _to_ft6d(c)
    return c


def _to_ft6d(c):
    x = 16 // c.elem_bytes
    nL, nR, H, S, D = c.K.shape
    K6 = c.K.reshape(nL, nR, H, S, D // x, x).transpose(0, 1, 2, 4, 3, 5).copy()
    return Cache(K6, c.V.copy(), c.layer_begin, c.req_begin, c.n_heads, c.max_seq, c.head_dim, LAYOUT_FT6D)


@pytest.mark.parametrize("layout", [LAYOUT_KV5D, LAYOUT_FT6D])
def test_pack_brute_equals_vector(layout):
    rng = np.random.default_rng(3)
    for _ in range(6):
        H, D, S = int(rng.integers(1, 4)), 8, int(rng.integers(4, 12))
        nL, nR = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        K = rng.integers(0, 1 << 16, (nL, nR, H, S, D), dtype=np.uint16)
        V = rng.integers(0, 1 << 16, (nL, nR, H, S, D), dtype=np.uint16)
        c = Cache(K, V, 5, 2, H, S, D)
        if layout == LAYOUT_FT6D:
            c = _to_ft6d(c)
        l0 = 5 + int(rng.integers(0, nL)); l1 = int(rng.integers(l0 + 1, 5 + nL + 1))
        r0 = 2 + int(rng.integers(0, nR)); r1 = int(rng.integers(r0 + 1, 2 + nR + 1))
        s0 = int(rng.integers(0, S)); s1 = int(rng.integers(s0 + 1, S + 1))
        reg = (l0, l1, r0, r1, s0, s1)
        wb, wv = pack(c, reg, "brute"), pack(c, reg, "vector")
        assert np.array_equal(wb, wv)
        d1, d2 = c.copy(), c.copy()
        for a in (d1.K, d1.V, d2.K, d2.V):
            a[...] = kvgen.SENTINEL
        unpack(d1, reg, wb, "brute")
        unpack(d2, reg, wv, "vector")
        assert np.array_equal(d1.K, d2.K) and np.array_equal(d1.V, d2.V)


@pytest.mark.parametrize("dst_layout", [LAYOUT_KV5D, LAYOUT_FT6D])
def test_uid_remap_c1_every_word_decodes_to_its_coordinate(dst_layout):
    """C1 toy (L2 H4 D16 b2, 32+8 positions, S 40 -> 64): after remapping region R, every
    destination word inside R decodes (uid) to exactly the global coordinate it sits at; every
    word outside R is still the sentinel; no poison crossed over."""
    L, B, H, S, D = 2, 2, 4, 40, 16
    box = (L, B, H, S, D)
    src = _uid_cache(0, L, 0, B, H, S, D, box, valid=(0, 36))
    dst = Cache(*kvgen.sentinel_cache(L, B, H, 64, D), 0, 0, H, 64, D)
    if dst_layout == LAYOUT_FT6D:
        dst = _to_ft6d(dst)
    reg = (0, 2, 1, 2, 3, 36)
    remap(src, dst, reg, "brute")
    for kv in (0, 1):
        lg = dst.logical(kv, 0, L, 0, B, 0, 64)    # [l][r][h][s][d]
        ll, rr, hh, ss, dd = np.meshgrid(*[np.arange(n) for n in lg.shape], indexing="ij")
        inside = (rr >= 1) & (ss >= 3) & (ss < 36)
        assert np.all(lg[~inside] == kvgen.SENTINEL)
        dk, dl, dr, dh, ds, dd_ = kvgen.uid_decode(lg[inside], box)
        assert np.all(dk == kv) and np.all(dl == ll[inside]) and np.all(dr == rr[inside])
        assert np.all(dh == hh[inside]) and np.all(ds == ss[inside]) and np.all(dd_ == dd[inside])
        assert not np.any(lg == kvgen.POISON)


def test_wire_order_is_layer_kv_request_head_pos_d():
    """Reading Q3: wire = [l][kv][r][h][s][d]. Decoding the uid of each wire word gives
    coordinates in exactly that row-major order."""
    L, B, H, S, D = 2, 2, 4, 40, 16
    box = (L, B, H, S, D)
    src = _uid_cache(0, L, 0, B, H, S, D, box)
    wire = pack(src, (0, 2, 0, 2, 32, 40), "brute")
    kv, l, r, h, s, d = kvgen.uid_decode(wire, box)
    exp = np.array(list(itertools.product(range(2), range(2), range(2), range(4), range(32, 40), range(16))))
    assert np.array_equal(np.stack([l, kv, r, h, s, d], 1), exp)


def test_fig6_positions_prompt_then_tokens(golden):
    """PAPER.md:119 / Fig. 6: a 4-word prompt fills positions [0,4) in every layer; each of the
    next 2 tokens updates one more position per layer. Stream prompt then each token to a host
    cache and check the filled set after each stream."""
    g = golden("scenario_rules.json")["fig6_positions"]
    p = g["prompt"]
    L, B, H, S, D = 3, 1, 2, 8, 8
    dev = Cache(*kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=6), 0, 0, H, S, D)
    host = Cache(*kvgen.sentinel_cache(L, B, H, S, D), 0, 0, H, S, D)
    regions = [(0, L, 0, B, 0, p)] + [(0, L, 0, B, oracle.token_position(p, t), oracle.token_position(p, t) + 1)
                                       for t in range(1, g["tokens"] + 1)]
    for reg, (lo, hi) in zip(regions, g["filled_after"]):
        remap(dev, host, reg)
        filled = ~np.all(host.K == kvgen.SENTINEL, axis=(0, 1, 2, 4))
        assert np.flatnonzero(filled).tolist() == list(range(lo, hi))
        # per-token update is 2 * L * B * H runs of D words (small, non-contiguous): PAPER.md:119
    assert np.array_equal(host.K[:, :, :, :p + 2], dev.K[:, :, :, :p + 2])


def test_round_trip_and_incremental_equals_bulk():
    """Stream-out to a host log then stream-in restores the cache;
    p-prompt then t per-token streams == one stream of [0, p+t)."""
    L, B, H, S, D, p, T = 4, 3, 2, 24, 8, 10, 5
    s = Setup([0, L], [0, B], S)
    src = {(0, 0): Cache(*kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=9), 0, 0, H, S, D)}
    inc = {(0, 0): Cache(*kvgen.sentinel_cache(L, B, H, S, D), 0, 0, H, S, D)}
    bulk = {(0, 0): Cache(*kvgen.sentinel_cache(L, B, H, S, D), 0, 0, H, S, D)}
    for lay in range(L):                                    # prompt, layer by layer (Opt 2)
        box = stream_out(src, s, s, (lay, lay + 1, 0, B, 0, p))
        stream_in(inc, s, s, (lay, lay + 1, 0, B, 0, p), box)
    for t in range(1, T + 1):
        q = oracle.token_position(p, t)
        stream(src, s, inc, s, (0, L, 0, B, q, q + 1))
    stream(src, s, bulk, s, (0, L, 0, B, 0, p + T))
    assert np.array_equal(inc[(0, 0)].K, bulk[(0, 0)].K) and np.array_equal(inc[(0, 0)].V, bulk[(0, 0)].V)
    exp = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=9, valid_pos=(0, p + T))
    for kv in (0, 1):
        got = bulk[(0, 0)].arr(kv)
        assert np.array_equal(got[:, :, :, :p + T], exp[kv][:, :, :, :p + T])
        assert np.all(got[:, :, :, p + T:] == kvgen.SENTINEL)


@pytest.mark.parametrize("psplit,tsplit", [
    ([0, 4, 8, 12], [0, 3, 7, 12]),
    ([0, 6, 12], [0, 5, 12]),
    ([0, 12], [0, 2, 4, 6, 8, 10, 12]),
])
@pytest.mark.parametrize("preq,treq", [([0, 4], [0, 2, 4]), ([0, 2, 4], [0, 4]), ([0, 4], [0, 4])])
def test_disaggregation_partition_invariance(psplit, tsplit, preq, treq):
    """north_star / PAPER.md:266: whatever the prompt partition and batch split, each token
    cache ends up equal to the single-machine logical KV (kvgen's definition) on [0,p) and
    sentinel beyond; the prompt caches are unchanged."""
    H, D, p, Sp, St, seed = 2, 8, 9, 12, 20, 33
    psetup, tsetup = Setup(psplit, preq, Sp), Setup(tsplit, treq, St)
    prompt = {}
    for i in range(psetup.n_stages):
        for u in range(psetup.n_micro):
            a, b = psplit[i], psplit[i + 1]
            c, d = preq[u], preq[u + 1]
            prompt[(i, u)] = Cache(*kvgen.kv5d_cache("hash", a, b - a, c, d - c, H, Sp, D, seed=seed,
                                                     valid_pos=(0, p)), a, c, H, Sp, D)
    snapshot = {k: (v.K.copy(), v.V.copy()) for k, v in prompt.items()}
    token = {}
    for j in range(tsetup.n_stages):
        for w in range(tsetup.n_micro):
            a, b = tsplit[j], tsplit[j + 1]
            c, d = treq[w], treq[w + 1]
            token[(j, w)] = Cache(*kvgen.sentinel_cache(b - a, d - c, H, St, D), a, c, H, St, D)
    scenarios.disaggregate(prompt, psetup, token, tsetup, p)
    for (j, w), tc in token.items():
        exp = kvgen.kv5d_cache("hash", tc.layer_begin, tc.n_layers, tc.req_begin, tc.n_reqs, H, St, D, seed=seed)
        for kv in (0, 1):
            assert np.array_equal(tc.arr(kv)[:, :, :, :p], exp[kv][:, :, :, :p])
            assert np.all(tc.arr(kv)[:, :, :, p:] == kvgen.SENTINEL)
    for k, (K, V) in snapshot.items():
        assert np.array_equal(prompt[k].K, K) and np.array_equal(prompt[k].V, V)


# ---------------------------------------------------------------------------------------------
# scenario rules (§4.2.2, §4.2.3)
# ---------------------------------------------------------------------------------------------
def test_swap_rules(golden):
    g = golden("scenario_rules.json")
    for ex in g["swap_rotation"]:
        assert oracle.swap_rotation(ex["x"], ex["N"]) == (ex["in"], ex["out"]), ex["cite"]
    for ex in g["swap_budget"]:
        assert oracle.swap_budget(ex["D"], ex["M"]) == (ex["host"], ex["device"]), ex["cite"]
    # one round touches every microbatch once per direction
    for N in range(2, 9):
        ins, outs = zip(*[oracle.swap_rotation(x, N) for x in range(N)])
        assert sorted(ins) == list(range(N)) and sorted(outs) == list(range(N))
    # transf_i volume = i * B * C, checked against an actual pack of the prefix
    H, D, B, i = 2, 8, 3, 7
    c = Cache(*kvgen.kv5d_cache("hash", 0, 1, 0, B, H, 16, D, seed=2), 0, 0, H, 16, D)
    C = 2 * H * D * 2
    assert pack(c, (0, 1, 0, B, 0, i)).nbytes == oracle.swap_in_bytes(i, B, C)


def test_ring_and_recovery_rules(golden):
    g = golden("scenario_rules.json")
    for ex in g["ring"]:
        assert oracle.ring_successor(ex["x"], ex["N"]) == ex["to"], ex["cite"]
    r = g["recovery_fig10"]
    assert [list(c) for c in oracle.recovery_copies(r["x"], r["N"])] == r["copies"], r["cite"]


def _write_token_factory(H, D, seed):
    def write(c, x, pos):
        for kv in (0, 1):
            blk = kvgen.logical_block("hash", kv, range(c.layer_begin, c.layer_begin + c.n_layers),
                                      range(c.req_begin, c.req_begin + c.n_reqs), H, [pos], D, seed)
            c.set_logical(kv, c.layer_begin, c.layer_begin + c.n_layers, c.req_begin,
                          c.req_begin + c.n_reqs, pos, pos + 1, blk)
    return write


@pytest.mark.parametrize("depth,rounds", [(3, 2), (4, 3), (5, 1)])
def test_swap_simulation_invariants(depth, rounds):
    """§4.2.2: after the rotation, each host arena holds the writer's words on [0, len_x) and the
    sentinel beyond; each swap-in moved the full prefix (log) and each swap-out one position; at
    most 2 microbatches are device resident."""
    L0, nL, b, H, S, D, p, seed = 3, 2, 2, 2, 16, 8, 5, 44
    host = {}
    for x in range(depth):
        K, V = kvgen.kv5d_cache("hash", L0, nL, x * b, b, H, S, D, seed=seed, valid_pos=(0, p))
        K[:, :, :, p:] = kvgen.SENTINEL
        V[:, :, :, p:] = kvgen.SENTINEL
        host[x] = Cache(K, V, L0, x * b, H, S, D)
    slots = [Cache(*kvgen.sentinel_cache(nL, b, H, S, D), L0, 0, H, S, D) for _ in range(2)]
    log = []
    seen = []

    def slot_holds_prefix(x, slot, n):
        # after each swap-in the slot equals the writer's words on [0, len)
        exp = kvgen.kv5d_cache("hash", L0, nL, x * b, b, H, S, D, seed=seed)
        for kv in (0, 1):
            assert np.array_equal(slot.arr(kv)[:, :, :, :n], exp[kv][:, :, :, :n]), (x, n)
        seen.append((x, n))
    length = scenarios.swap_simulate(host, slots, p, rounds, _write_token_factory(H, D, seed), log,
                                     after_swap_in=slot_holds_prefix)
    assert len(seen) == len([e for e in log if e[0] == "in"]) > 0
    for x in range(depth):
        assert length[x] == p + rounds
        exp = kvgen.kv5d_cache("hash", L0, nL, x * b, b, H, S, D, seed=seed)
        for kv in (0, 1):
            a = host[x].arr(kv)
            assert np.array_equal(a[:, :, :, :length[x]], exp[kv][:, :, :, :length[x]])
            assert np.all(a[:, :, :, length[x]:] == kvgen.SENTINEL)
    ins = [e for e in log if e[0] == "in"]
    outs = [e for e in log if e[0] == "out"]
    assert all(e[2] == 0 for e in ins)                   # swap-in moves the whole prefix (Q8)
    assert all(e[3] - e[2] == 1 for e in outs)           # swap-out moves only the step delta
    assert len(outs) == depth * rounds                   # every step's delta reaches the host
    resident = {0}
    for e in log[1:]:
        if e[0] == "out":
            resident.discard(e[1])
        else:
            resident.add(e[1])
        assert len(resident) <= 2


def test_ring_replication_and_recovery():
    """§4.2.3: replica of stage x at (x+1)%N equals x's cache on [0, p+t) after each step; after
    a failure of x (its own cache and the replica it hosts wiped), the two recovery copies restore
    both exactly."""
    N, Ls, b, H, S, D, p, T, seed = 4, 2, 2, 2, 16, 8, 6, 3, 55
    own, rep = {}, {}
    for x in range(N):
        own[x] = Cache(*kvgen.kv5d_cache("hash", x * Ls, Ls, 0, b, H, S, D, seed=seed, valid_pos=(0, p)),
                       x * Ls, 0, H, S, D)
        px = (x - 1) % N
        rep[x] = Cache(*kvgen.sentinel_cache(Ls, b, H, S, D), px * Ls, 0, H, S, D)
    scenarios.ring_step(own, rep, lambda x: (x * Ls, x * Ls + Ls, 0, b, 0, p))   # prompt replica (Q13)
    write = _write_token_factory(H, D, seed)
    for t in range(1, T + 1):
        q = oracle.token_position(p, t)
        for x in range(N):
            write(own[x], x, q)
        scenarios.ring_step(own, rep, lambda x: (x * Ls, x * Ls + Ls, 0, b, q, q + 1))
        for x in range(N):
            y = (x + 1) % N
            assert np.array_equal(rep[y].K[:, :, :, :q + 1], own[x].K[:, :, :, :q + 1])
            assert np.array_equal(rep[y].V[:, :, :, :q + 1], own[x].V[:, :, :, :q + 1])
    before_own = own[1].copy()
    before_rep = rep[1].copy()
    for a in (own[1].K, own[1].V, rep[1].K, rep[1].V):
        a[...] = kvgen.SENTINEL
    scenarios.recover(1, own, rep, p + T)
    n = p + T   # everything replicated up to the last acked step; beyond it was never written
    for a, bfr in ((own[1].K, before_own.K), (own[1].V, before_own.V), (rep[1].K, before_rep.K),
                   (rep[1].V, before_rep.V)):
        assert np.array_equal(a[:, :, :, :n], bfr[:, :, :, :n])
        assert np.all(a[:, :, :, n:] == kvgen.SENTINEL)


def test_kvgen_hash_is_splitmix64():
    """kvgen's generator is the published splitmix64 finaliser: known first outputs of the
    splitmix64 sequence seeded with 0 (state += golden gamma, then the finaliser)."""
    # Reference values of splitmix64 with state 0: next() returns mix(0x9E3779B97F4A7C15), ...
    got = kvgen.splitmix64(np.array([0, 0x9E3779B97F4A7C15], dtype=np.uint64))
    assert int(got[0]) == 0xE220A8397B1DCDAF
    assert int(got[1]) == 0x6E789E6AA1B965F4


def test_log_form_swap_round_trip_equals_definition():
    """Host log form (C4): the prompt as one chunk, then one chunk per token step
    appended; unpacking the log rebuilds exactly kvgen's words on [0, p+T) and nothing else."""
    L, B, H, S, D, p, T = 3, 2, 2, 24, 8, 7, 6
    src = Cache(*kvgen.kv5d_cache("hash", 4, L, 2, B, H, S, D, seed=13), 4, 2, H, S, D)
    prompt = pack(src, (4, 4 + L, 2, 2 + B, 0, p))
    steps = [pack(src, (4, 4 + L, 2, 2 + B, p + t, p + t + 1)) for t in range(T)]
    dst = Cache(*kvgen.sentinel_cache(L, B, H, S, D), 4, 2, H, S, D)
    unpack(dst, (4, 4 + L, 2, 2 + B, 0, p), prompt)
    from oracle.kvstream import unpack_chunks
    unpack_chunks(dst, (4, 4 + L, 2, 2 + B, p, p + 1), np.concatenate(steps), T, 1)
    exp = kvgen.kv5d_cache("hash", 4, L, 2, B, H, S, D, seed=13)
    for kv in (0, 1):
        assert np.array_equal(dst.arr(kv)[:, :, :, :p + T], exp[kv][:, :, :, :p + T])
        assert np.all(dst.arr(kv)[:, :, :, p + T:] == kvgen.SENTINEL)
    # chunks of 2 positions with pos_step 3 leave every third position untouched
    dst2 = Cache(*kvgen.sentinel_cache(L, B, H, S, D), 4, 2, H, S, D)
    log2 = np.concatenate([pack(src, (4, 4 + L, 2, 2 + B, 3 * k, 3 * k + 2)) for k in range(4)])
    unpack_chunks(dst2, (4, 4 + L, 2, 2 + B, 0, 2), log2, 4, 3, mode="brute")
    filled = ~np.all(dst2.K == kvgen.SENTINEL, axis=(0, 1, 2, 4))
    assert np.flatnonzero(filled).tolist() == [0, 1, 3, 4, 6, 7, 9, 10]


# ---------------------------------------------------------------------------------------------
# tensor-parallel head split (NEXT-4; "tensor parallelism inside a stage")
# ---------------------------------------------------------------------------------------------
def test_route_tp_2_to_4_splits_each_head_group_in_two():
    """Same stages, TP 2 -> 4 over 8 heads: each source head group [0,4), [4,8) splits into two
    destination groups (the head analogue of SPEC.md:376's depth split)."""
    src = Setup([0, 4], [0, 2], 16, head_bounds=[0, 4, 8])
    dst = Setup([0, 4], [0, 2], 16, head_bounds=[0, 2, 4, 6, 8])
    ps = route(src, dst, (0, 4, 0, 2, 0, 5), 8, 16, 2)
    assert [(p.src_tp, p.dst_tp, p.head_begin, p.head_end) for p in ps] == \
        [(0, 0, 0, 2), (0, 1, 2, 4), (1, 2, 4, 6), (1, 3, 6, 8)]
    assert all(p.bytes == 2 * 4 * 2 * 5 * 2 * 16 * 2 for p in ps)
    assert [p.src_wire_off for p in ps] == [0, ps[0].bytes, 0, ps[2].bytes]
    with pytest.raises(ValueError):                       # one side split, the other not
        route(src, Setup([0, 4], [0, 2], 16), (0, 4, 0, 2, 0, 5), 8, 16, 2)
    with pytest.raises(MappingError):                     # heads not held
        route(src, dst, (0, 4, 0, 2, 0, 5, 0, 9), 8, 16, 2)


@pytest.mark.parametrize("seed", range(25))
def test_route_tp_brute_force_coverage(seed):
    rng = random.Random(700 + seed)
    L, R, Hn = rng.randint(1, 6), rng.randint(1, 5), rng.randint(1, 9)
    mk = lambda n, k: _random_bounds(rng, 0, n, rng.randint(1, min(n, k)))
    src = Setup(mk(L, 3), mk(R, 2), 32, head_bounds=mk(Hn, 4))
    dst = Setup(mk(L, 3), mk(R, 2), 32, head_bounds=mk(Hn, 4))
    ps = route(src, dst, (0, L, 0, R, 3, 7), Hn, 8, 2)
    for l in range(L):
        for r in range(R):
            for h in range(Hn):
                cov = [p for p in ps if p.layer_begin <= l < p.layer_end and p.req_begin <= r < p.req_end
                       and p.head_begin <= h < p.head_end]
                assert len(cov) == 1
                p = cov[0]
                assert src.head_bounds[p.src_tp] <= h < src.head_bounds[p.src_tp + 1]
                assert dst.head_bounds[p.dst_tp] <= h < dst.head_bounds[p.dst_tp + 1]
    assert sum(p.bytes for p in ps) == 2 * L * R * 4 * Hn * 8 * 2


@pytest.mark.parametrize("sh,th", [([0, 6], [0, 3, 6]), ([0, 2, 4, 6], [0, 3, 6]), ([0, 3, 6], [0, 1, 2, 3, 4, 5, 6])])
def test_disaggregation_with_tp_resplit_equals_definition(sh, th):
    """Prompt pipeline TP degree != token pipeline TP degree (NEXT-4): every token shard equals
    kvgen's words for its own layers, requests and HEADS."""
    H, D, p, S, seed = 6, 8, 5, 9, 41
    ps_, ts_ = Setup([0, 2, 4], [0, 2], S, head_bounds=sh), Setup([0, 3, 4], [0, 2], S, head_bounds=th)
    prompt, token = {}, {}
    for i in range(ps_.n_stages):
        for t in range(ps_.n_tp):
            a, b, h0, h1 = ps_.layer_bounds[i], ps_.layer_bounds[i + 1], sh[t], sh[t + 1]
            K, V = kvgen.kv5d_cache("hash", a, b - a, 0, 2, h1 - h0, S, D, seed=seed, head_begin=h0)
            prompt[(i, 0, t)] = Cache(K, V, a, 0, h1 - h0, S, D, head_begin=h0)
    for j in range(ts_.n_stages):
        for t in range(ts_.n_tp):
            a, b, h0, h1 = ts_.layer_bounds[j], ts_.layer_bounds[j + 1], th[t], th[t + 1]
            token[(j, 0, t)] = Cache(*kvgen.sentinel_cache(b - a, 2, h1 - h0, S, D), a, 0, h1 - h0, S, D,
                                     head_begin=h0)
    stream(prompt, ps_, token, ts_, (0, 4, 0, 2, 0, p))
    for (j, _, t), c in token.items():
        exp = kvgen.kv5d_cache("hash", c.layer_begin, c.n_layers, 0, 2, c.n_heads, S, D, seed=seed,
                               head_begin=c.head_begin)
        for kv in (0, 1):
            assert np.array_equal(c.arr(kv)[:, :, :, :p], exp[kv][:, :, :, :p])
            assert np.all(c.arr(kv)[:, :, :, p:] == kvgen.SENTINEL)


def test_ft6d_key_layout_matches_fastertransformer_indexing():
    """NEXT-1: in the 6-D key layout word (l,r,h,s,d) sits at [l][r][h][d//x][s][d%x], x = 16/e
    (16-byte packets); the oracle's FT6D cache agrees element by element with that formula."""
    L, B, H, S, D = 2, 2, 3, 6, 16
    K, V = kvgen.kv5d_cache("uid", 0, L, 0, B, H, S, D, box=(L, B, H, S, D))
    K6 = kvgen.as_ft6d_key(K)
    c = Cache(K6, V, 0, 0, H, S, D, layout=LAYOUT_FT6D)
    for l, r, h, s_, d in itertools.product(range(L), range(B), range(H), range(S), range(D)):
        assert K6[l, r, h, d // 8, s_, d % 8] == K[l, r, h, s_, d]
        assert c.K[c.word_index(0, l, r, h, s_, d)] == K[l, r, h, s_, d]
    assert np.array_equal(pack(c, (0, L, 0, B, 1, 5), "brute"),
                          pack(Cache(K, V, 0, 0, H, S, D), (0, L, 0, B, 1, 5), "vector"))


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.uint32, np.uint64])
def test_ft6d_packet_width_is_16_bytes_for_every_word_size(dtype):
    """NEXT-1 for opaque words of 1/2/4/8 bytes: a FasterTransformer key packet is 16 BYTES, so it
    holds x = 16/e words; the element (l,r,h,s,d) sits at [l][r][h][d//x][s][d%x]. K6 is built here
    by explicit loops from that definition (independent of kvgen.as_ft6d_key and of the oracle)."""
    e = np.dtype(dtype).itemsize
    x = 16 // e
    L, B, H, S, D = 2, 2, 2, 5, 2 * x
    K = np.arange(L * B * H * S * D, dtype=np.uint64).astype(dtype).reshape(L, B, H, S, D)
    V = (K + 1).astype(dtype)
    K6 = np.zeros((L, B, H, D // x, S, x), dtype)
    for l, r, h, s_, d in itertools.product(range(L), range(B), range(H), range(S), range(D)):
        K6[l, r, h, d // x, s_, d % x] = K[l, r, h, s_, d]
    c6 = Cache(K6, V, 0, 0, H, S, D, layout=LAYOUT_FT6D)
    for l, r, h, s_, d in itertools.product(range(L), range(B), range(H), range(S), range(D)):
        assert c6.K[c6.word_index(0, l, r, h, s_, d)] == K[l, r, h, s_, d]
    reg = (0, L, 0, B, 1, 4)
    assert np.array_equal(pack(c6, reg, "brute"), pack(Cache(K, V, 0, 0, H, S, D), reg, "vector"))
