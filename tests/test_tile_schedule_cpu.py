"""The K > 1 similarity passes' local-first tile schedule (sim_kernel.cu `pair_items` /
`decode_item`, SimParams::local_first), restated here: every pair takes a contiguous share of the
group-ordered own-tile list and a share of the remote-tile list that makes its total the balanced
floor(T (p+1) / P) - floor(T p / P), running the remote share in reverse. The host launches at
most T / 2 pairs. Checked for every rank of the shapes the passes see: each (group, column tile)
exactly once, pair loads within one tile of each other, no negative remote share."""
import pytest

TILE = 256


def schedule(n_rb, n_jt, rank, rows_per_rank, n_pairs_cap=74):
    col_lo = rank * rows_per_rank
    jt_lo = (col_lo + TILE - 1) // TILE
    n_loc = max(0, min((rank + 1) * rows_per_rank // TILE, n_jt) - jt_lo)
    n_tiles = 2 * n_rb * n_jt
    pairs = max(1, min(n_pairs_cap, n_tiles // 2))   # pair_grid(n_items / 2)
    own = 2 * n_rb * n_loc
    out = []
    for p in range(pairs):
        c_lo, c_hi = n_tiles * p // pairs, n_tiles * (p + 1) // pairs
        t_lo = own * p // pairs
        n_own = own * (p + 1) // pairs - t_lo
        rem_lo = c_lo - t_lo
        count = max(c_hi - c_lo, n_own)
        assert count - n_own >= 0
        items = []
        for item in range(count):
            if item < n_own:
                u = t_lo + item
                grp, jt = u // n_loc, jt_lo + u % n_loc
            else:
                n_rem = n_jt - n_loc
                v = rem_lo + (count - 1 - item)
                grp, r = v // n_rem, v % n_rem
                jt = r if r < jt_lo else r + n_loc
            items.append((grp, jt, item < n_own))
        out.append(items)
    return out, jt_lo, n_loc


@pytest.mark.parametrize("B,K", [(512, 2), (1024, 4), (2560, 2), (4096, 4), (5120, 2), (5120, 4), (5120, 8),
                                 (8192, 8), (16384, 4)])
def test_local_first_schedule_covers_every_tile_once(B, K):
    rows = B // K
    n_jt = (B + TILE - 1) // TILE
    n_rb = (rows + TILE - 1) // TILE
    for rank in range(K):
        pairs, jt_lo, n_loc = schedule(n_rb, n_jt, rank, rows)
        seen = [(g, j) for items in pairs for g, j, _ in items]
        assert sorted(seen) == [(g, j) for g in range(2 * n_rb) for j in range(n_jt)], (B, K, rank)
        loads = [len(items) for items in pairs]
        assert max(loads) - min(loads) <= 1, (B, K, rank, loads)
        for items in pairs:   # own tiles (caller's slice) strictly before remote ones
            flags = [own for _, _, own in items]
            assert flags == sorted(flags, reverse=True)
            for g, j, own in items:
                assert own == (jt_lo <= j < jt_lo + n_loc)
