"""bench.py host logic on CPU: the C5 library's shard cuts (shard_bounds over
the virtual C2 x 100 buffer) are newline-aligned, cover every byte once and
match shard_bounds on the materialised buffer."""

import numpy as np

import bench
import synth
from paper_2404_19391_b200 import shard


def test_virtual_bounds_match_shard_bounds():
    c2 = synth.generate("aromatic", 3000, 2024)
    reps = 7
    full = np.tile(c2, reps)
    for world in (1, 2, 3, 4, 8):
        cuts = bench.virtual_bounds(c2, reps, world)
        flat = [k * c2.size + off for k, off in cuts]
        assert flat == shard.shard_bounds(full, world), world
        for c in flat[1:-1]:
            assert full[c - 1] == 0x0A
