"""CPU checks of the z-line table's coverage arithmetic (sl_step.cu:
zt_reach_kernel / zt_cover_kernel, sl_device.cuh: zt_covered), restated in
Python: a brick whose feet move at most D cells must cover every table node
its stencils read, so that the per-foot lookup only fails for feet beyond
the bound (the lookup itself keeps the result exact either way)."""
import math

import numpy as np
import pytest

B = 4  # kZtBrick


def floor_div(a, b):  # sl_step.cu floor_div
    return a // b


def packed_reach(cells):  # zt_reach_kernel: ceil(D) << 8 | floor(D)
    return (math.ceil(cells) << 8) | math.floor(cells)


def cover_offsets(r):  # zt_cover_kernel
    rn, rp = r >> 8, r & 0xFF
    return (floor_div(-rn - 1, B), floor_div(B + 1 + rp, B)), (floor_div(-rn, B), floor_div(B + rp, B))


@pytest.mark.parametrize("cells", [0.0, 0.3, 1.0, 1.9, 2.0, 2.9, 3.0, 4.5, 6.49, 7.0, 11.2])
def test_cover_contains_every_stencil_table_node(cells):
    (lo, hi), (loz, hiz) = cover_offsets(packed_reach(cells))
    rng = np.random.default_rng(int(cells * 100))
    for local in range(B):  # node position inside its brick (brick 10, nodes 40..43)
        i = 10 * B + local
        for delta in np.concatenate([[-cells, cells, 0.0], rng.uniform(-cells, cells, 200)]):
            c = math.floor(i + delta)  # locate_cell of the foot (before clamping)
            xs = range(c - 1, c + 3)   # x / y table nodes of the 4x4x4 stencil
            zs = range(c, c + 2)       # z table nodes (planes cz, cz + 1)
            assert all(10 + lo <= x // B <= 10 + hi for x in xs), (cells, local, delta)
            assert all(10 + loz <= z // B <= 10 + hiz for z in zs), (cells, local, delta)


def test_packed_reach_is_monotone():
    """atomicMax on the packed value keeps the largest displacement bound."""
    vals = np.linspace(0.0, 12.0, 2401)
    packed = [packed_reach(v) for v in vals]
    assert all(a <= b for a, b in zip(packed, packed[1:]))


def test_covered_lookup_spans_at_most_two_bricks_per_axis():
    """zt_covered reads the bricks of (c - 1) and (c + 2) per x/y axis and of
    c and c + 1 along z: every table node of the stencil lies in one of them."""
    for c in range(1, 60):
        bx = {x // B for x in range(c - 1, c + 3)}
        assert bx <= {(c - 1) // B, (c + 2) // B}
        bz = {z // B for z in range(c, c + 2)}
        assert bz <= {c // B, (c + 1) // B}
