"""CPU model of the FFMA kernel's minimal-padding reduce-scatter
(csrc/ffma_ws.cuh ws_reduce_scatter): the same level structure, send/keep
selection, jb / nreal / dup bookkeeping, run on symbolic partials.  Every
real partial j of every column group must land in exactly one writing lane
and be the sum of exactly the 32/LANES_T lanes of its group -- including
odd counts, where a padded slot's index coincides with another lane's real
partial (the case the nreal bookkeeping exists for)."""

import pytest


def model(NR, LT):
    lanes = 32
    v = {l: [{(l, j)} for j in range(NR)] for l in range(lanes)}
    cur = NR; o = LT
    state = {l: dict(jb=0, dup=False, nreal=NR) for l in range(lanes)}
    while o < 32:
        new = {}
        if cur > 1:
            half = (cur + 1) // 2
            for l in range(lanes):
                up = bool(l & o); p = l ^ o
                def hi(x, i): return v[x][i + half] if i + half < cur else set()
                out = []
                for i in range(half):
                    keep = hi(l, i) if up else v[l][i]
                    recv = hi(p, i) if up else v[p][i]
                    out.append(keep | recv)
                new[l] = out
                st = state[l]
                if up: st['jb'] += half; st['nreal'] = max(st['nreal'] - half, 0)
                else: st['nreal'] = min(st['nreal'], half)
            cur = half
        else:
            for l in range(lanes):
                new[l] = [v[l][0] | v[l ^ o][0]]
                if l & o: state[l]['dup'] = True
        v = new; o *= 2
    got = {}
    for l in range(lanes):
        st = state[l]
        if st['dup']: continue
        for i in range(cur):
            j = st['jb'] + i
            if i < st['nreal'] and j < NR:
                assert (l % LT, j) not in got, (NR, LT, j)
                got[(l % LT, j)] = (l, v[l][i])
    assert sorted(got) == [(t, j) for t in range(LT) for j in range(NR)], (NR, LT, sorted(got))
    for (t, j), (l, sset) in got.items():
        bad = [x for x in sset if x[1] != j]
        # lanes of the same k-group: same (l % LT) (tq) -> LT cosets
        lanes_in = {x[0] for x in sset}
        if bad or len(lanes_in) != 32 // LT or any((x % LT) != (l % LT) for x in lanes_in):
            return False
    return True


@pytest.mark.parametrize("NR", [1, 2, 3, 5, 7, 11, 13, 21, 22, 31, 32, 33, 44])
@pytest.mark.parametrize("LT", [1, 2, 4, 8])
def test_reduce_scatter_places_every_partial_once(NR, LT):
    assert model(NR, LT)
