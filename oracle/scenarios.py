"""Scenario oracles -- TEST INFRASTRUCTURE ONLY (see oracle/kvstream.py header).

Each scenario is a sequence of the plain byte relocations of kvstream.py in the order the paper
describes; the GPU tests replay the same sequence through the C ABI and compare final states.

  swap_simulate     -- §4.2.2 microbatch swapping, PAPER.md:270-272 (Fig. 9), reading Q10.
  ring_step         -- §4.2.3 replication, worker x -> (x+1)%N per token.
  recover           -- §4.2.3 steps 1-2 of recovery.
  disaggregate      -- §4.2.1 prompt->token hand-off with split/merge.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Tuple

from .kvstream import (Cache, Setup, remap, ring_successor, stream, swap_rotation,
                       token_position, recovery_copies)


def swap_simulate(host: Dict[int, Cache], slots: List[Cache], prompt_len: int, rounds: int,
                  write_token: Callable[[Cache, int, int], None], log: list | None = None,
                  after_swap_in: Callable[[int, Cache, int], None] | None = None):
    """One stage of a depth-D pipeline (D = len(host) >= 3) with two device slots.

    host[x] is microbatch x's host arena in mirror form (same layout, holds [0, len_x));
    initially every arena holds its prompt [0, prompt_len) (streamed out layer by layer during the
    prompt pass). Events are processed in pipeline order x = 0..D-1, ``rounds``
    times. For the event "microbatch x runs token step t":
      (b) the writer fills position p+t-1 of x in its slot,
      (c) swap-out: the delta of (x-1)%D -- the one position its last step wrote -- goes to its
          host arena (only the step's update moves out),
      (d) swap-in: the whole prefix [0, len) of (x+1)%D (PAPER.md:572 transf_i = i*B*C) goes into
          the slot (x-1)%D just released; (c) completes before (d) overwrites that slot (Q10).
    Before the first event microbatch 0 is swapped into slot 0; after the last event the final
    delta is swapped out. Mutates host/slots; returns {x: len_x}.
    ``log`` (optional) receives ('in'|'out', x, pos_begin, pos_end, slot) tuples (the regions
    actually moved); ``after_swap_in`` (optional) is called as (x, slot seen as x's cache, len_x)
    right after each swap-in, so a test can check the slot's contents at that moment.
    """
    D = len(host)
    if D < 3:
        raise ValueError("two-slot rotation needs D >= 3 (Q9)")
    c = host[0]
    L0, L1 = c.layer_begin, c.layer_begin + c.n_layers
    length = {x: prompt_len for x in range(D)}
    steps_done = {x: 0 for x in range(D)}
    slot_of = {0: 0}

    def swap_in(x, slot):
        reg = (L0, L1, host[x].req_begin, host[x].req_begin + host[x].n_reqs, 0, length[x])
        remap(host[x], relabel(slots[slot], host[x].req_begin), reg)
        slot_of[x] = slot
        if log is not None:
            log.append(("in", x, reg[4], reg[5], slot))
        if after_swap_in is not None:
            after_swap_in(x, relabel(slots[slot], host[x].req_begin), length[x])

    def swap_out(x):
        pos = length[x] - 1
        reg = (L0, L1, host[x].req_begin, host[x].req_begin + host[x].n_reqs, pos, pos + 1)
        remap(relabel(slots[slot_of[x]], host[x].req_begin), host[x], reg)
        if log is not None:
            log.append(("out", x, reg[4], reg[5], slot_of[x]))

    swap_in(0, 0)
    last = None
    for t in range(1, rounds + 1):
        for x in range(D):
            xin, xout = swap_rotation(x, D)
            pos = token_position(prompt_len, t)
            write_token(relabel(slots[slot_of[x]], host[x].req_begin), x, pos)
            steps_done[x] += 1
            length[x] = prompt_len + steps_done[x]
            if steps_done[xout] > 0 and xout in slot_of:
                swap_out(xout)
                free = slot_of.pop(xout)
            else:
                free = 1 - slot_of[x]
            if not (t == rounds and x == D - 1):
                swap_in(xin, free)
            last = x
    swap_out(last)
    return length


def relabel(c: Cache, req_begin: int) -> Cache:
    """The same arrays seen as holding requests [req_begin, +n): a device slot holds whichever
    microbatch is resident ("2*M GB in GPU memory")."""
    return Cache(c.K, c.V, c.layer_begin, req_begin, c.n_heads, c.max_seq, c.head_dim, c.layout)


def ring_step(own: Dict[int, Cache], replica: Dict[int, Cache], region_of: Callable[[int], tuple]):
    """Every stage x streams region_of(x) of its own cache into the replica store it keeps at
    (x+1)%N. replica[y] holds stage (y-1)%N's layers."""
    n = len(own)
    for x in range(n):
        remap(own[x], replica[ring_successor(x, n)], region_of(x))


def recover(x: int, own: Dict[int, Cache], replica: Dict[int, Cache], pos_end: int):
    """Recovery copies for failed worker x: (1) replica of x held at (x+1)%N -> x's
    own cache, (2) own cache of (x-1)%N -> the replica store at x. Positions [0, pos_end)."""
    n = len(own)
    (a, _, _), (b, _, _) = recovery_copies(x, n)
    ox = own[x]
    remap(replica[a], ox, (ox.layer_begin, ox.layer_begin + ox.n_layers, ox.req_begin,
                           ox.req_begin + ox.n_reqs, 0, pos_end))
    ob = own[b]
    remap(ob, replica[x], (ob.layer_begin, ob.layer_begin + ob.n_layers, ob.req_begin,
                           ob.req_begin + ob.n_reqs, 0, pos_end))


def disaggregate(prompt: Dict[Tuple[int, int], Cache], psetup: Setup,
                 token: Dict[Tuple[int, int], Cache], tsetup: Setup, prompt_len: int):
    """Prompt KV of every layer and request, positions [0,p), prompt pipeline -> token pipeline
    (PAPER.md:266), split/merged by the route."""
    region = (psetup.layer_bounds[0], psetup.layer_bounds[-1], psetup.req_bounds[0],
              psetup.req_bounds[-1], 0, prompt_len)
    return stream(prompt, psetup, token, tsetup, region)
