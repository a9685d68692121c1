"""CPU model of the long-line colouring (csrc/zs_ll.cuh ll_colour + ll_umin):
closing events cut into segments, each run from a guessed entry lc[] (no
closes), then passes in which a segment compares its left neighbour's exit --
normalised at u, the earliest opening before the segment of a ring closing in
it -- with what it assumed, runs again if they differ, and otherwise passes
the neighbour's entries through for the colours it did not touch; exits are
normalised at U, the minimum u of every later segment.  Segments run in
"parallel" (each pass reads the previous pass's exits).  The model must give
the colours of the reference's _color_intervals (smiles.py:163-183) on random
ring soups, with tiny segments so that crossing rings and long passthrough
chains are common.
"""

import random

import pytest

NCOL = 100


def reference_colours(events):
    """events: list of ring ids in line order -> colour per event (smiles.py:140-183)."""
    open_at, intervals = {}, []
    for i, rid in enumerate(events):
        if rid in open_at:
            intervals.append((open_at.pop(rid), i))
        else:
            open_at[rid] = i
    assert not open_at
    assigned, col = [], {}
    for o, c in sorted(intervals, key=lambda iv: iv[1]):
        used = {k for o2, c2, k in assigned if o2 < c and o < c2}
        k = 0
        while k in used:
            k += 1
        assigned.append((o, c, k))
        col[o] = col[c] = k
    return [col[i] for i in range(len(events))]


def model_colours(events, seg):
    n = len(events)
    part, last = [], {}
    for i, rid in enumerate(events):  # ll_pair: a close's partner is the nearest earlier same id
        if rid in last:
            part.append(last.pop(rid))
        else:
            part.append(-1)
            last[rid] = i
    nseg = (n + seg - 1) // seg
    colour = [None] * n

    def run(s, lc_in):
        a, b = s * seg, min(n, (s + 1) * seg)
        lc = dict(lc_in)  # colour -> last close (absent: -1)
        touched = set()
        for e in range(a, b):
            o = part[e]
            if o < 0:
                continue
            k = 0
            while lc.get(k, -1) > o:
                k += 1
            lc[k] = e
            touched.add(k)
            colour[e] = colour[o] = k
        return lc, touched

    u = [min([part[e] for e in range(s * seg, min(n, (s + 1) * seg)) if part[e] >= 0] + [s * seg])
         for s in range(nseg)]
    U = [min(u[s + 1:], default=1 << 30) for s in range(nseg)]  # ll_umin

    def norm(lc, t):
        return {k: v for k, v in lc.items() if v > t}

    assumed = [dict() for _ in range(nseg)]
    exits, touched = [], []
    for s in range(nseg):  # pass 0: guessed entries
        lc, t = run(s, {})
        exits.append(lc)
        touched.append(t)
    for _ in range(4 * nseg + 4):  # fix passes (each reads the previous pass's exits)
        prev = [dict(x) for x in exits]
        changed = False
        for s in range(nseg):
            incoming = prev[s - 1] if s else {}
            if u[s] < s * seg and norm(incoming, u[s]) != assumed[s]:
                assumed[s] = norm(incoming, u[s])
                lc, touched[s] = run(s, incoming)
            else:
                lc = {k: v for k, v in incoming.items() if k not in touched[s]}
                lc.update({k: exits[s][k] for k in touched[s] if k in exits[s]})
            new = norm(lc, U[s])
            if new != exits[s]:
                exits[s] = new
                changed = True
        if not changed:
            return colour
    raise AssertionError("the fix passes did not settle")


def soup(rng, n_events, width):
    ev, open_, free = [], [], list(range(1, 100))
    while len(ev) < n_events:
        if open_ and (len(open_) >= width or rng.random() < 0.5):
            rid = open_.pop(rng.randrange(len(open_)))
            free.append(rid)
        else:
            rid = free.pop(rng.randrange(len(free)))
            open_.append(rid)
        ev.append(rid)
    return ev + open_


@pytest.mark.parametrize("seed", range(12))
def test_segmented_colouring_equals_reference(seed):
    rng = random.Random(seed)
    for _ in range(8):
        ev = soup(rng, rng.randint(1, 400), rng.choice([1, 2, 3, 5, 12, 40]))
        want = reference_colours(ev)
        for seg in (1, 2, 3, 7, 16, 128):
            assert model_colours(ev, seg) == want, (seed, seg)
