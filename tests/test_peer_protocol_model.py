"""Model check of the JACC_GRAPH_P2P peer protocol (csrc/peer.cuh), on CPU.

The GPU tests can only run world 2 as two time-sliced contexts on one GPU;
here the protocol's LOGIC (epochs counted on the device, flag-in-data small
allreduce double-buffered by epoch parity, the ready/data handshake of the
all-gather, the grid ticket) is executed at world 2-4 under thousands of
random interleavings of every rank's blocks, each shared-memory access being
a scheduling point.  Each rank runs an SPMD program for several epochs --
the bench's step (fused allreduce, fused all-gather, a kernel reading the
gathered buffer), the same allreduce back to back, or the N-body chain
(all-gather, reader, all-gather, ...) -- and every value read is checked
against the epoch it must belong to.  Memory is sequentially consistent in
the model: the fences and the PTX ordering argument are not modelled (they
are argued in peer.cuh); what is checked is that no schedule can deadlock,
read a stale or a future epoch's data, or overwrite data still being read.

The model has teeth: removing the parity double-buffering or the ready
handshake (each a plausible mistake) is detected.
"""
import random

import pytest


class Deadlock(Exception):
    pass


class Rank:
    def __init__(self, world, slots, n):
        self.data = [[0] * world for _ in range(slots)]    # data[slot][src]
        self.ready = [[0] * world for _ in range(slots)]   # ready[slot][src]
        self.count = [0] * slots
        self.ticket = [0] * slots
        # LL staging: stage[slot][parity][src][i] = (tag, value)
        self.stage = [[[[(0, 0)] * n for _ in range(world)] for _ in range(2)] for _ in range(slots)]
        self.recv = [None] * (world * n)                    # all-gather receive buffer


def run_model(world, epochs, seed, n=3, blocks=2, parity=True, ready=True, program="suite"):
    """Returns the list of errors found (empty = correct)."""
    rnd = random.Random(seed)
    W = [Rank(world, 2, n) for _ in range(world)]
    errors = []
    AR, AG = 0, 1   # slots: allreduce, all-gather

    def val(r, e, i):            # rank r's contribution to the allreduce, epoch e
        return 1000 * e + 10 * r + i

    def pos(r, e, i):            # rank r's i-th position produced in epoch e
        return (r, e, i)

    # ---- kernels (generators yielding at every shared access) ----------
    def k_allreduce(r):
        """block_allreduce: one block; LL words (tag = epoch) into row [r] of
        every rank's staging (parity e & 1), poll own rows, sum in rank order."""
        me = W[r]
        e = me.count[AR] + 1
        yield
        p = (e & 1) if parity else 0
        for i in range(n):
            for q in range(world):
                W[q].stage[AR][p][r][i] = (e, val(r, e, i))
                yield
        for i in range(n):
            acc = 0
            for q in range(world):
                while me.stage[AR][p][q][i][0] != e:
                    if me.stage[AR][p][q][i][0] > e:
                        errors.append(f"rank {r} epoch {e}: allreduce row {q} overwritten by epoch "
                                      f"{me.stage[AR][p][q][i][0]}")
                        return
                    yield "wait"
                acc += me.stage[AR][p][q][i][1]
                yield
            want = sum(val(q, e, i) for q in range(world))
            if acc != want:
                errors.append(f"rank {r} epoch {e}: allreduce[{i}] = {acc}, want {want}")
        me.count[AR] = e

    def k_allgather_blocks(r):
        """Fused N-body finish + all-gather: block 0 publishes ready; every
        block waits for each receiver's ready, stores its slice there; grid
        ticket; the last block publishes data and waits for every rank's."""
        me = W[r]
        e = me.count[AG] + 1   # read by every block before the last bumps it
        per = (n + blocks - 1) // blocks

        def block(b):
            yield
            if b == 0:
                for q in range(world):
                    W[q].ready[AG][r] = e
                    yield
            for q in range(world):
                if q != r and ready:
                    while me.ready[AG][q] < e:
                        yield "wait"
                for i in range(b * per, min(n, (b + 1) * per)):
                    W[q].recv[r * n + i] = pos(r, e, i)
                    yield
            me.ticket[AG] += 1
            last = me.ticket[AG] == blocks
            yield
            if not last:
                return
            me.ticket[AG] = 0
            for q in range(world):
                W[q].data[AG][r] = e
                yield
            me.count[AG] = e
            for q in range(world):
                while me.data[AG][q] < e:
                    yield "wait"
        return [block(b) for b in range(blocks)]

    def k_reader(r):
        """The next step's partial kernel: reads every gathered position."""
        me = W[r]
        e = me.count[AG]
        for i in range(world * n):
            got = me.recv[i]
            want = pos(i // n, e, i % n)
            if got != want:
                errors.append(f"rank {r} epoch {e}: recv[{i}] = {got}, want {want}")
                return
            yield

    # ---- per-rank stream: kernels in order, a kernel = a set of blocks ----
    def stream(r):
        for _ in range(epochs):
            if program != "nbody":
                yield [k_allreduce(r)]
            if program != "allreduce":
                yield k_allgather_blocks(r)
                yield [k_reader(r)]
            # "suite": allreduce + all-gather + reader per epoch;
            # "allreduce": the same allreduce back to back (a graph of
            #   histogram -> allreduce executed repeatedly);
            # "nbody": the N-body chain -- all-gather, then the next step's
            #   partial kernel reading it, nothing else in between

    streams = [stream(r) for r in range(world)]
    running = [next(s) for s in streams]           # current kernel's live blocks per rank
    waits = 0
    while any(running):
        cand = [(r, j) for r in range(world) for j in range(len(running[r] or []))]
        if not cand:
            break
        r, j = rnd.choice(cand)
        try:
            y = next(running[r][j])
            waits = waits + 1 if y == "wait" else 0
            if waits > 200000:
                raise Deadlock(f"seed {seed}: no progress")
        except StopIteration:
            running[r].pop(j)
            if not running[r]:
                running[r] = next(streams[r], None)
        if errors:
            break
    return errors


@pytest.mark.parametrize("program", ["suite", "allreduce", "nbody"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_protocol_correct_under_random_schedules(world, program):
    for seed in range(300 if world == 2 else 150):
        errs = run_model(world, epochs=4, seed=seed, program=program)
        assert not errs, errs[:3]


def test_model_detects_missing_parity():
    """Single-buffered LL rows: a fast rank's next epoch overwrites a row a
    slow rank has not read yet -- some schedule must expose it."""
    found = any(run_model(2, epochs=4, seed=s, parity=False, program="allreduce") for s in range(400))
    assert found


def test_model_detects_missing_ready_handshake():
    """Storing into a peer's gathered buffer without waiting for its ready:
    the peer's reader sees the next epoch's positions in some schedule."""
    found = any(run_model(2, epochs=4, seed=s, ready=False, program="nbody") for s in range(400))
    assert found
