"""Random-schedule model of the mbarrier protocol of fp_pack_bulk_crc
(pack.cu): producer warp (TMA G2S fill, FULL wait, hand-off of tile i to
its CRC group, then EMPTY wait + FREE + refill for tile i - 1), two LSU
warps, kGroups groups of CRC warps. mbarrier semantics as PTX defines them: a phase completes when its pending arrivals
and transaction bytes reach zero; try_wait.parity(P) succeeds iff the current
phase's parity differs from P. The model checks that every schedule finishes
(no deadlock) and that a CRC warp only ever reads the tile it was handed.
The first two-group design (CRC warps testing FULL[s] themselves) fails here
as it hung on the GPU (test_first_design_fails)."""
import random

import pytest

STAGES = 3  # kBcStages


class Bar:
    def __init__(self, count):
        self.count, self.pend, self.tx, self.phase = count, count, 0, 0

    def arrive(self, tx=0):
        self.tx += tx
        self.pend -= 1
        self._check()

    def complete_tx(self, b):
        self.tx -= b
        self._check()

    def _check(self):
        if self.pend == 0 and self.tx == 0:
            self.phase += 1
            self.pend = self.count

    def test(self, parity):  # mbarrier.try_wait.parity
        return (self.phase & 1) != parity


def run(nt, groups, warps, seed, old=False):
    """One random schedule of a CTA with nt tiles; 'ok', 'deadlock' or 'wrong tile'."""
    rnd = random.Random(seed)
    full = [Bar(1 + 2) for _ in range(STAGES)]        # producer expect_tx + 2 LSU warps
    empty = [Bar(warps) for _ in range(STAGES)]       # the CRC warps of the tile's group
    freeb = [Bar(1) for _ in range(STAGES)]
    cfull = [Bar(1) for _ in range(2 * groups)]       # [group][j & 1]
    tma = []                                          # G2S in flight: (stage, tile)
    in_stage = [None] * STAGES
    bad = []

    def producer():
        def fill(i):
            s = i % STAGES
            full[s].arrive(tx=1)
            tma.append((s, i))
        for i in range(min(nt, STAGES)):
            fill(i)
            yield
        for i in range(nt):
            s = i % STAGES
            while not full[s].test((i // STAGES) & 1):
                yield
            cfull[(i % groups) * 2 + ((i // groups) & 1)].arrive()
            yield
            if old:             # first design: drain tile i, refill its stage
                if i + STAGES < nt:
                    while not empty[s].test((i // STAGES) & 1):
                        yield
                    freeb[s].arrive()
                    fill(i + STAGES)
                    yield
            elif i:             # drain tile i - 1 behind tile i's hand-off
                p = i - 1
                while not empty[p % STAGES].test((p // STAGES) & 1):
                    yield
                if p + STAGES < nt:
                    freeb[p % STAGES].arrive()
                    fill(p + STAGES)
                    yield
        if not old and nt:
            while not empty[(nt - 1) % STAGES].test(((nt - 1) // STAGES) & 1):
                yield

    def lsu():
        for i in range(nt):
            s = i % STAGES
            if i >= STAGES:
                while not freeb[s].test((i // STAGES - 1) & 1):
                    yield
            full[s].arrive()
            yield

    def crc(g):
        for j, i in enumerate(range(g, nt, groups)):
            s = i % STAGES
            if old:
                if groups > 1 and i >= STAGES:
                    while not full[s].test((i // STAGES - 1) & 1):
                        yield
                while not full[s].test((i // STAGES) & 1):
                    yield
            else:
                while not cfull[g * 2 + (j & 1)].test((j >> 1) & 1):
                    yield
            if in_stage[s] != i:
                bad.append((i, in_stage[s]))
            empty[s].arrive()
            yield

    alive = [producer(), lsu(), lsu()] + [crc(g) for g in range(groups) for _ in range(warps)]
    for _ in range(200000):
        if not alive and not tma:
            return "wrong tile" if bad else "ok"
        if tma and (not alive or rnd.random() < 0.3):
            s, i = tma.pop(rnd.randrange(len(tma)))
            in_stage[s] = i
            full[s].complete_tx(1)
            continue
        a = rnd.choice(alive)
        try:
            next(a)
        except StopIteration:
            alive.remove(a)
    return "deadlock"


@pytest.mark.parametrize("groups", [1, 2])
def test_protocol_never_deadlocks(groups):
    for nt in range(1, 12):
        for seed in range(60):
            assert run(nt, groups, 2, seed) == "ok", (nt, groups, seed)


def test_first_design_fails():
    assert any(run(8, 2, 2, seed, old=True) != "ok" for seed in range(20))
