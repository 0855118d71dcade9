"""Tiling value types, descriptors and grid queries (SURVEY §8 a1–a4) against
hand-derived answers from the reference's definitions
(/root/reference/pkg/src/unimul/tiling.py:18-221, cli.py:140-165).  The C++
planner's owner query is checked against this module in test_capi.py.  CPU only."""

import random

import pytest

from paper_2510_08874_b200 import tiling as T
from paper_2510_08874_b200.cli import resolve_partition
from paper_2510_08874_b200.errors import ConfigError
from paper_2510_08874_b200.tiling import Bounds2D, GridShape, Mapping, PartitionSpec, Range, Shape2D, TileIdx


def test_range_is_half_open_and_validated():
    r = Range(3, 7)
    assert len(r) == 4 and str(r) == "[3,7)" and r.shift(-3) == Range(0, 4)
    assert len(Range(5, 5)) == 0
    for lo, hi in ((-1, 2), (4, 3)):
        with pytest.raises(ValueError):
            Range(lo, hi)


def test_bounds_shape_area_contains():
    b = Bounds2D(Range(2, 6), Range(1, 4))
    assert b.shape == Shape2D(4, 3) and b.area == 12
    assert b.contains(Bounds2D(Range(2, 3), Range(3, 4)))
    assert not b.contains(Bounds2D(Range(1, 3), Range(1, 2)))
    assert b.contains(Bounds2D(Range(6, 6), Range(1, 1)))       # empty at the edge


def test_partition_spec_rejects_empty_shapes():
    with pytest.raises(ConfigError):
        PartitionSpec(Shape2D(0, 4), Shape2D(1, 1))
    with pytest.raises(ConfigError):
        PartitionSpec(Shape2D(4, 4), Shape2D(2, 0))


@pytest.mark.parametrize("p,grid", [(1, (1, 1)), (2, (1, 2)), (4, (2, 2)), (6, (2, 3)), (7, (1, 7)),
                                    (8, (2, 4)), (12, (3, 4)), (16, (4, 4)), (18, (3, 6))])
def test_most_square_grid(p, grid):
    assert T.most_square_grid(p) == Shape2D(*grid)


def test_descriptors():
    g = Shape2D(10, 7)
    assert T.row_block(g, 4) == PartitionSpec(Shape2D(3, 7), Shape2D(4, 1))
    assert T.col_block(g, 4) == PartitionSpec(Shape2D(10, 2), Shape2D(1, 4))
    assert T.block_2d(g, 6) == PartitionSpec(Shape2D(5, 3), Shape2D(2, 3))
    # more ranks than rows: bands of at least one row, trailing ranks own nothing
    assert T.row_block(Shape2D(3, 5), 8).tile_shape == Shape2D(1, 5)
    # cfg5's A at p=8: 2d = 8192 x 4096 tiles on a 2 x 4 grid
    assert T.block_2d(Shape2D(16384, 16384), 8) == PartitionSpec(Shape2D(8192, 4096), Shape2D(2, 4))
    assert resolve_partition("2d", Shape2D(16384, 16384), 8) == T.block_2d(Shape2D(16384, 16384), 8)
    assert resolve_partition("row", g, 4) == T.row_block(g, 4)
    assert resolve_partition("col", g, 4) == T.col_block(g, 4)
    assert resolve_partition("misaligned", g, 12) == PartitionSpec(Shape2D(3, 4), Shape2D(3, 4))
    assert resolve_partition("custom:2:3:1:4:cyclic", g, 4) == PartitionSpec(Shape2D(2, 3), Shape2D(1, 4),
                                                                             Mapping.BLOCK_CYCLIC)
    with pytest.raises(ConfigError):
        resolve_partition("custom:2", g, 4)


def test_grid_and_ragged_tile_bounds():
    part = PartitionSpec(Shape2D(4, 3), Shape2D(2, 2))
    g = Shape2D(10, 7)
    assert T.grid_shape(part, g) == GridShape(3, 3)
    assert T.tile_bounds(part, g, TileIdx(0, 0)) == Bounds2D(Range(0, 4), Range(0, 3))
    assert T.tile_bounds(part, g, TileIdx(2, 2)) == Bounds2D(Range(8, 10), Range(6, 7))   # clipped
    for bad in (TileIdx(3, 0), TileIdx(0, 3), TileIdx(-1, 0)):
        with pytest.raises(IndexError):
            T.tile_bounds(part, g, bad)
    # the tiles partition the matrix exactly
    cells = set()
    for t in T.grid_shape(part, g).tiles():
        b = T.tile_bounds(part, g, t)
        cells |= {(r, c) for r in range(b.rows.lo, b.rows.hi) for c in range(b.cols.lo, b.cols.hi)}
    assert len(cells) == g.rows * g.cols


def test_overlapping_tiles_row_major_and_empty():
    part = PartitionSpec(Shape2D(4, 3), Shape2D(1, 1))
    g = Shape2D(10, 7)
    got = T.overlapping_tiles(part, g, Bounds2D(Range(3, 9), Range(2, 4)))
    assert got == [TileIdx(0, 0), TileIdx(0, 1), TileIdx(1, 0), TileIdx(1, 1), TileIdx(2, 0), TileIdx(2, 1)]
    assert T.overlapping_tiles(part, g, Bounds2D(Range(4, 8), Range(3, 6))) == [TileIdx(1, 1)]
    assert T.overlapping_tiles(part, g, Bounds2D(Range(5, 5), Range(0, 7))) == []


def test_intersect_canonical_empty():
    assert T.intersect(Range(2, 8), Range(5, 12)) == Range(5, 8)
    assert T.intersect(Range(2, 4), Range(6, 9)) == Range(6, 6)      # disjoint: [lo, lo) at the larger lo
    assert T.intersect(Range(6, 9), Range(2, 4)) == Range(6, 6)
    a = Bounds2D(Range(0, 4), Range(0, 4))
    assert T.intersect_bounds(a, Bounds2D(Range(2, 6), Range(5, 7))) == Bounds2D(Range(2, 4), Range(5, 5))


def test_owner_block_and_cyclic():
    # BLOCK: 5 x 5 tiles on a 2 x 2 grid -> ceil(5/2) = 3 x 3 tiles per rank block
    part = PartitionSpec(Shape2D(1, 1), Shape2D(2, 2))
    grid = GridShape(5, 5)
    assert [T.owner_of(part, grid, TileIdx(i, 0), 4) for i in range(5)] == [0, 0, 0, 2, 2]
    assert [T.owner_of(part, grid, TileIdx(0, j), 4) for j in range(5)] == [0, 0, 0, 1, 1]
    assert T.owner_of(part, grid, TileIdx(4, 4), 4) == 3
    cyc = PartitionSpec(Shape2D(1, 1), Shape2D(2, 2), Mapping.BLOCK_CYCLIC)
    assert [T.owner_of(cyc, grid, TileIdx(i, i), 4) for i in range(5)] == [0, 3, 0, 3, 0]
    assert T.owner_of(cyc, grid, TileIdx(3, 2), 4) == 2
    with pytest.raises(ConfigError):
        T.owner_of(part, grid, TileIdx(0, 0), 8)
    with pytest.raises(IndexError):
        T.owner_of(part, grid, TileIdx(5, 0), 4)


def test_block_owner_covers_every_rank_when_grid_divides():
    rng = random.Random(5)
    for _ in range(50):
        pr, pc = rng.randint(1, 4), rng.randint(1, 4)
        gr, gc = pr * rng.randint(1, 3), pc * rng.randint(1, 3)
        part = PartitionSpec(Shape2D(1, 1), Shape2D(pr, pc))
        owners = [T.owner_of(part, GridShape(gr, gc), t, pr * pc) for t in GridShape(gr, gc).tiles()]
        assert sorted(set(owners)) == list(range(pr * pc))
        assert all(owners.count(r) == (gr // pr) * (gc // pc) for r in range(pr * pc))
