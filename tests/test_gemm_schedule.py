"""The CTA-pair GEMM's stream-K schedule (gemm_tcgen05.cu: sk_plan / sk_item),
restated in Python and checked for the properties the kernel relies on:
every (tile, k-block) computed exactly once, one finisher per split tile that
reads exactly the partial slots its earlier pieces wrote, in k order, and
every partial piece is its pair's FIRST stream-K item (so a finisher never
waits on a pair that is itself waiting: no wait chains, no deadlock)."""

import random

import pytest

KBK = 64
SKW = 32 * 128


def sk_plan(M, N, K, W):
    tiles = ((M + 255) // 256) * ((N + 255) // 256)
    nk = (K + KBK - 1) // KBK
    plan = dict(dp_tiles=tiles, units=0, pieces=1, slots=0, tiles=tiles, nk=nk)
    if M <= 128 or tiles % W == 0 or tiles * nk < 8 * W:
        return plan
    full = tiles // W
    dp = (full - 1) * W if full >= 1 else 0
    units = (tiles - dp) * nk
    lmin = units // W
    if lmin < 4:
        return plan
    pieces = (nk + lmin - 1) // lmin + 1
    plan.update(dp_tiles=dp, units=units, pieces=pieces, slots=(tiles - dp) * (pieces - 1))
    return plan


def sk_item(pl, c, W, i):
    nk = pl["nk"]
    dp = pl["dp_tiles"]
    ndp = (dp - c + W - 1) // W if c < dp else 0
    if i < ndp:
        return dict(tile=c + i * W, kb0=0, kb1=nk, kind=0, slot=0, npart=0)
    U = pl["units"]
    if U == 0:
        return None
    u0, u1 = c * U // W, (c + 1) * U // W
    if u0 >= u1:
        return None
    t = (u1 - 1) // nk - (i - ndp)
    if t < u0 // nk:
        return None
    tb = t * nk
    kb0, kb1 = max(u0, tb) - tb, min(u1, tb + nk) - tb
    first = ((tb + 1) * W - 1) // U
    slot = t * (pl["pieces"] - 1)
    if kb1 < nk:
        return dict(tile=dp + t, kb0=kb0, kb1=kb1, kind=1, slot=slot + (c - first), npart=0)
    if kb0 == 0:
        return dict(tile=dp + t, kb0=kb0, kb1=kb1, kind=0, slot=slot, npart=0)
    return dict(tile=dp + t, kb0=kb0, kb1=kb1, kind=2, slot=slot, npart=c - first)


def check(M, N, K, W):
    pl = sk_plan(M, N, K, W)
    cover = {}
    partial_pieces = {}     # slot -> (tile, kb0, kb1)
    finishers = {}
    for c in range(W):
        i = 0
        ndp = (pl["dp_tiles"] - c + W - 1) // W if c < pl["dp_tiles"] else 0
        while True:
            it = sk_item(pl, c, W, i)
            if it is None:
                break
            for kb in range(it["kb0"], it["kb1"]):
                key = (it["tile"], kb)
                assert key not in cover, f"{key} computed twice"
                cover[key] = c
            if it["kind"] == 1:
                assert i == ndp, "a partial piece must be its pair's first stream-K item"
                assert 0 <= it["slot"] < pl["slots"] and it["slot"] not in partial_pieces
                assert it["slot"] - (it["tile"] - pl["dp_tiles"]) * (pl["pieces"] - 1) < pl["pieces"] - 1
                partial_pieces[it["slot"]] = (it["tile"], it["kb0"], it["kb1"])
            elif it["kind"] == 2:
                assert it["tile"] not in finishers
                finishers[it["tile"]] = it
            i += 1
    assert len(cover) == pl["tiles"] * pl["nk"], "every (tile, k-block) exactly once"
    for tile, f in finishers.items():
        slots = [f["slot"] + p for p in range(f["npart"])]
        assert all(s in partial_pieces and partial_pieces[s][0] == tile for s in slots)
        kbs = [partial_pieces[s][1:] for s in slots] + [(f["kb0"], f["kb1"])]
        assert kbs[0][0] == 0 and all(a[1] == b[0] for a, b in zip(kbs, kbs[1:])), "pieces in k order"
        del_slots = set(slots)
        for s in del_slots:
            partial_pieces.pop(s)
    assert not partial_pieces, "every partial piece is consumed by its tile's finisher"
    return pl


@pytest.mark.parametrize("N,K", [(6144, 2048), (2048, 2048), (8192, 2048), (2048, 8192), (50272, 2048)])
def test_schedule_at_model_shapes(N, K):
    pl = check(2048, N, K, 74)
    if N != 8192 or K != 2048:
        assert pl["units"] > 0          # these shapes leave a partial wave: stream-K is on


def test_schedule_random_shapes():
    rng = random.Random(3)
    for _ in range(300):
        M = rng.choice([256, 512, 1024, 2048, 3000, 4096, 8192])
        N = rng.randrange(64, 20000, 8)
        K = rng.randrange(64, 9000, 8)
        W = rng.choice([1, 2, 7, 66, 74])
        check(M, N, K, W)
