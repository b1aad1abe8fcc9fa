"""Host-side model of the mbarrier protocol of the C5 apply kernel (k_c5.cu k_c5_apply):
the producer / MMA / converter / epilogue roles, written as coroutines that wait and arrive on
the same barriers in the same program order as the kernel, run under every interleaving a
round-robin scheduler produces. Checks, for the shipped ring depths and a range of per-CTA unit
counts, that (1) the protocol cannot deadlock and (2) every parity wait is released by exactly
the phase it waits for -- an mbarrier parity wait cannot tell phase k from phase k + 2, so a
waiter that could run two phases ahead would read stale data without any error."""
import pytest


ARRIVALS = [0]


class Barrier:
    def __init__(self, count=1):
        self.count, self.pending, self.phases = count, 0, 0

    def arrive(self):
        ARRIVALS[0] += 1
        self.pending += 1
        if self.pending == self.count:
            self.pending = 0
            self.phases += 1


class ABA(Exception):
    pass


def wait(b, idx):
    """Coroutine: wait for completion number idx of b through its parity (as try_wait.parity)."""
    while (b.phases % 2) == (idx & 1):  # hardware: released iff the current phase parity differs
        yield "wait"
    if b.phases != idx + 1:
        raise ABA(f"released at {b.phases} completions while waiting for completion #{idx}")


def apply_roles(n_my, S, NLO, bepi=True, nacc=2, bi=False, ring=16, upb=4):
    """nacc: accumulators = B sets (unit i uses slot i % nacc); the W~ staging ring stays 2 deep.
    bi: the default fused kernel with B-image records (k_c5.cu BI >= 1): a setup-group role publishes
    units in batches of `upb` (the first at once, every other one after the next batch's conversion)
    into a ring of `ring` records that it may only rewrite once the apply has consumed them
    (units_built, set by epilogue warp 8 after accfull); thread 128 bulk-copies unit j's image into B
    set j % nacc (bready completes by the copy's bytes) once the setup has published it."""
    B = lambda c=1: Barrier(c)
    yfull, yfree = [B() for _ in range(S)], [B() for _ in range(S)]
    afull, afree = [B() for _ in range(NLO)], [B() for _ in range(NLO)]
    bready, accfull, tfree = [B() for _ in range(nacc)], [B() for _ in range(nacc)], [B() for _ in range(nacc)]
    wfull, wfree = [B() for _ in range(2)], [B() for _ in range(2)]
    G = 4 * n_my
    st8 = {"ready": 0, "built": 0}  # the kernel's shared-memory counters units_ready / units_built

    def setup():  # fused setup group (bi): batch k = units 4k .. 4k + nv - 1
        nb = (n_my + upb - 1) // upb
        for k in range(nb):
            j0, nv = upb * k, min(upb, n_my - upb * k)
            if k > 0:
                st8["ready"] = j0  # publish_prev after this batch's conversion
            while st8["built"] < j0 + nv - ring:  # ring_wait before the batch's record writes
                yield "wait"
            yield "step"
            if k == 0 and nv < n_my:
                st8["ready"] = nv  # the first batch at once
        if n_my > 0:
            st8["ready"] = n_my

    def issue_b(j):  # spin on units_ready, then the image copy completes bready
        while st8["ready"] <= j:
            yield "wait"
        bready[j % nacc].arrive()

    def producer():
        def issue_w(i):
            if i >= 2:
                yield from wait(wfree[i & 1], (i >> 1) - 1)
            wfull[i & 1].arrive()  # TMA completes
        first = True
        for gg in range(G):
            st = gg % S
            if not bepi and gg & 3 == 0:  # BEPI: the B builder stages the W~ records itself
                if first:
                    first = False
                    yield from issue_w(0)
                    if n_my > 1:
                        yield from issue_w(1)
                if (gg >> 2) + 2 < n_my:
                    yield from issue_w((gg >> 2) + 2)
            if gg >= S:
                yield from wait(yfree[st], gg // S - 1)
            yfull[st].arrive()
            yield "step"

    def mma():
        for i in range(n_my):
            b = i % nacc
            yield from wait(bready[b], i // nacc)
            if i >= nacc:
                yield from wait(tfree[b], i // nacc - 1)
            for c in range(4):
                gg = 4 * i + c
                lb = gg % NLO
                yield from wait(afull[lb], gg // NLO)
                afree[lb].arrive()
                if c == 3:
                    accfull[b].arrive()
                yield "step"

    def build_b(i):
        yield from wait(wfull[i & 1], i >> 1)

    def converters():
        for i in range(n_my):
            b = i % nacc
            if not bepi:
                if i >= nacc:
                    yield from wait(accfull[b], i // nacc - 1)
                yield from build_b(i)
                bready[b].arrive()
                wfree[i & 1].arrive()
            for c in range(4):
                gg = 4 * i + c
                st, lb = gg % S, gg % NLO
                yield from wait(yfull[st], gg // S)
                if gg >= NLO:
                    yield from wait(afree[lb], gg // NLO - 1)
                afull[lb].arrive()
                yfree[st].arrive()
                yield "step"

    def epilogue():  # warps 4-7 (and the B builder with BEPI); warps 8-9 share the tfree barrier sync
        def stage_w(i):  # BEPI: thread 128 issues the W~ TMA of unit i into stage i & 1 (completes at once)
            wfull[i & 1].arrive()
        if bi:
            for j in range(min(nacc, n_my)):
                yield from issue_b(j)
            for i in range(n_my):
                b = i % nacc
                yield from wait(accfull[b], i // nacc)
                st8["built"] = i + 1  # warp 8 (not held by thread 128's spin below)
                if i + nacc < n_my:
                    yield from issue_b(i + nacc)
                tfree[b].arrive()
                yield "step"
            return
        if bepi:
            for i0 in range(min(2, n_my)):
                stage_w(i0)
            for j in range(min(nacc, n_my)):
                yield from build_b(j)
                bready[j].arrive()
                if j + 2 < n_my:
                    stage_w(j + 2)
        for i in range(n_my):
            b = i % nacc
            yield from wait(accfull[b], i // nacc)
            if bepi and i + nacc < n_my:
                yield from build_b(i + nacc)
                bready[b].arrive()
                if i + nacc + 2 < n_my:
                    stage_w(i + nacc + 2)
            tfree[b].arrive()
            yield "step"

    return [producer(), mma(), converters(), epilogue()] + ([setup()] if bi else [])


def run(roles, max_rounds=200000):
    alive = list(roles)
    for _ in range(max_rounds):
        before = ARRIVALS[0]
        progressed = False
        for r in list(alive):
            try:
                if next(r) == "step":
                    progressed = True
            except StopIteration:
                alive.remove(r)
                progressed = True
        if not alive:
            return True
        if not progressed and ARRIVALS[0] == before:
            # a full round in which every live role only re-polled: with no TMA/MMA latency left to
            # model, nothing can change any more
            return False
    return False


@pytest.mark.parametrize("S,NLO", [(6, 4), (4, 2), (8, 4), (7, 4), (5, 2)])
@pytest.mark.parametrize("bepi,nacc", [(True, 2), (False, 2), (True, 3)])
@pytest.mark.parametrize("n_my", [0, 1, 2, 3, 4, 5, 7, 8, 9, 13, 74])
def test_apply_protocol_no_deadlock_no_aba(S, NLO, bepi, nacc, n_my):
    assert run(apply_roles(n_my, S, NLO, bepi, nacc)), "protocol deadlocks"


@pytest.mark.parametrize("S,NLO", [(5, 2), (6, 4)])
@pytest.mark.parametrize("n_my", [0, 1, 2, 3, 4, 5, 7, 8, 9, 13, 16, 17, 21, 33, 74])
@pytest.mark.parametrize("ring", [16, 8])
def test_apply_protocol_b_images(S, NLO, n_my, ring):
    """The default C5 kernel (B-image records, setup group in the loop): no deadlock, no ABA."""
    assert run(apply_roles(n_my, S, NLO, bepi=True, nacc=2, bi=True, ring=ring)), "protocol deadlocks"


def test_model_detects_a_ring_too_small():
    """The checker itself: a ring shorter than one setup batch plus the apply's lookahead deadlocks
    (the setup group waits for slots the apply can only free after the records it waits for)."""
    assert not run(apply_roles(13, 5, 2, bepi=True, nacc=2, bi=True, ring=4))


def test_model_detects_a_two_phase_runaway():
    """The checker itself: a waiter two phases ahead of a barrier is reported (the hazard that
    made the slot-ring setup kernel hang before each worker warp owned its slot)."""
    b = Barrier()

    def early_waiter():
        yield from wait(b, 1)  # waits for the 2nd completion while the 1st has not happened

    with pytest.raises(ABA):
        next(early_waiter())
