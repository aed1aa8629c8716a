"""Model check of the face-exchange protocol of the mid-size resident leapfrog (csrc/mid.cu), on
the CPU: compute-sanitizer is closed on the GPU pool, so the protocol's safety argument is
checked here over many random interleavings of an abstract model of one launch (tags only).

* CTAs on an nby x nbz grid with the j-1 / k-1 / j+1 / k+1 neighbours of mid_box.
* Each CTA owns, per slot (2, by epoch parity t & 1), four regions of tagged lines: JM, KM (its
  e faces, read by the j-1 / k-1 neighbours) and JP, KP (its h faces, read by j+1 / k+1).
* Epoch 0 publishes JP, KP with tag 0 into slot 0.  Epoch t >= 1 is an e-half (t odd: stage the
  j-1 neighbour's JP and the k-1 neighbour's KP of slot (t-1)&1, then publish JM, KM into slot
  t&1) or an h-half (t even: stage the j+1 neighbour's JM and the k+1 neighbour's KM, publish
  JP, KP).
* Staging polls each needed line until it carries tag t-1 (exact match, as mid_stage); with the
  barrier every line read of an epoch completes before the CTA's first store of that epoch (the
  __syncthreads after mid_stage); stores are interleaved line by line with every other CTA's
  actions in random order.
A protocol error can only show as a poll that never completes (its line was overwritten by a
newer epoch before it was read): the model reports a deadlock.  The second test removes the
barrier and finds such deadlocks, so the model is sharp enough to see the race it rules out."""
import random

import pytest


def _neighbours(c, nby, nbz):
    cy, cz = c % nby, c // nby
    return (c - 1 if cy > 0 else -1, c - nby if cz > 0 else -1,
            c + 1 if cy + 1 < nby else -1, c + nby if cz + 1 < nbz else -1)


def simulate(nby, nbz, epochs, lines, rng, barrier=True):
    """Run one launch; returns True, raises AssertionError on a deadlock or a bad overwrite."""
    ncta = nby * nbz
    tag = [[[[None] * lines for _ in range(4)] for _ in range(2)] for _ in range(ncta)]
    nb = [_neighbours(c, nby, nbz) for c in range(ncta)]
    t_of = [0] * ncta
    reads = [[] for _ in range(ncta)]     # pending line reads of the current epoch
    stores = [[] for _ in range(ncta)]    # pending line stores of the current epoch

    def stores_of(c, t):
        slot = t & 1
        regs = ((0, nb[c][0]), (1, nb[c][1])) if t % 2 == 1 else ((2, nb[c][2]), (3, nb[c][3]))
        return [(slot, r, l) for r, n in regs if n >= 0 for l in range(lines)]

    def start(c, t):
        t_of[c] = t
        if t == 0:
            reads[c] = []
            stores[c] = [(0, r, l) for r, n in ((2, nb[c][2]), (3, nb[c][3])) if n >= 0 for l in range(lines)]
            return
        sidx = (t - 1) & 1
        need = ((nb[c][0], 2), (nb[c][1], 3)) if t % 2 == 1 else ((nb[c][2], 0), (nb[c][3], 1))
        reads[c] = [(n, sidx, r, l) for n, r in need if n >= 0 for l in range(lines)]
        stores[c] = stores_of(c, t)

    for c in range(ncta):
        start(c, 0)
    while any(t_of[c] <= epochs for c in range(ncta)):
        actions = []
        for c in range(ncta):
            if t_of[c] > epochs:
                continue
            t = t_of[c]
            for w in reads[c]:
                if tag[w[0]][w[1]][w[2]][w[3]] == t - 1:
                    actions.append((c, "read", w))
            if stores[c] and (not barrier or not reads[c]):
                actions.append((c, "store", None))
            if not reads[c] and not stores[c]:
                actions.append((c, "next", None))
        if not actions:
            raise AssertionError(f"deadlock at epochs {t_of}: a line overwritten before it was read")
        c, kind, w = rng.choice(actions)
        t = t_of[c]
        if kind == "read":
            reads[c].remove(w)
        elif kind == "store":
            slot, r, l = stores[c].pop(rng.randrange(len(stores[c])))
            assert tag[c][slot][r][l] in (None, t - 2), "a line overwritten out of epoch order"
            tag[c][slot][r][l] = t
        else:
            start(c, t + 1)
    return True


@pytest.mark.parametrize("nby,nbz", [(2, 1), (1, 3), (2, 2), (3, 2), (4, 3)])
def test_mid_exchange_protocol_never_deadlocks(nby, nbz):
    rng = random.Random(1000 * nby + nbz)
    for _ in range(80):
        assert simulate(nby, nbz, epochs=14, lines=2, rng=rng)


def test_without_the_staging_barrier_the_model_finds_the_race():
    """Stores allowed before the epoch's reads finish: a neighbour can run two epochs ahead and
    overwrite a line still to be read -- some interleaving deadlocks."""
    rng = random.Random(7)
    failures = 0
    for _ in range(300):
        try:
            simulate(3, 2, epochs=14, lines=2, rng=rng, barrier=False)
        except AssertionError:
            failures += 1
    assert failures > 0
