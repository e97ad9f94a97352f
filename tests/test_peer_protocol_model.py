"""Model check of the fused-halo (F1) IPC flag protocol of csrc/mfc.cu (peer_wait /
peer_signal), on CPU.

The device side cannot run here, so this executes the protocol's host-visible logic --
the same counters and slot arithmetic as the C++ -- for R ranks under many random
interleavings of their stream operations, and checks what the protocol must guarantee:

* no deadlock;
* every ghost read sees the neighbours' most recent write of that buffer (q, S1 or S2)
  in program order -- never older, never newer data;
* a rank writes a neighbour's buffer only after the neighbour has finished every earlier
  read of that buffer (the q -> S1 -> S2 -> q rotation of the RK stages);
* a signal never lands on a slot the receiver has not consumed yet (3 slots suffice:
  neighbours are at most one operation apart);
* the flag values a step uses are the same in every step (what makes a captured CUDA
  graph of a step replayable).

Programs follow the library's call patterns: mfc_halo_exchange (wait e-1, write, signal
e, wait e), mfc_rhs (an exchange, then one more operation that only signals), and RK3
steps (three operations, each waiting for the previous one of the neighbours)."""
import random

import pytest


Q, S1, S2 = 0, 1, 2                           # the registered state and the stage buffers


class Rank:
    def __init__(self, r, nbrs):
        self.r = r
        self.nbrs = nbrs                          # [face] -> neighbour rank
        self.flags = [[0, 0, 0] for _ in nbrs]    # [face][slot], written by the neighbour
        self.epoch = 0                            # operations completed (signalled)
        self.waited = 0                           # neighbour operations consumed
        self.reads_done = set()                   # operations whose ghost reads finished
        self.ghost = [[None, None, None] for _ in nbrs]   # [face][buffer] -> writer's op
        self.actions = []
        self.ops = {}                             # op index -> (reads, writes)


def build_program(rank, calls):
    """Expand the call sequence into the atomic stream operations of mfc.cu: operation e
    waits for the neighbours' e-1 (peer_wait), reads the ghosts of one buffer, writes the
    neighbours' ghosts of another (the stage result), signals e (peer_signal)."""
    acts = []
    e = 0

    def op(reads, writes, post_wait=False):
        nonlocal e
        e += 1
        rank.ops[e] = (reads, writes)
        acts.append(("wait", e - 1))
        if reads is not None:
            acts.append(("read", e))
        if writes is not None:
            acts.append(("write", e))
        acts.append(("signal", e))
        if post_wait:                             # exchange_fused's trailing wait
            acts.append(("wait", e))

    for c in calls:
        if c == "exchange":                       # my boundary layers -> neighbours' q ghosts
            op(None, Q, post_wait=True)
        elif c == "rhs":                          # exchange, then the sweeps read q's ghosts
            op(None, Q, post_wait=True)
            op(Q, None)
        elif c == "step":                         # q -> S1 -> S2 -> q
            op(Q, S1)
            op(S1, S2)
            op(S2, Q)
    rank.actions = acts


def enabled(ranks, me):
    a = me.actions[0]
    if a[0] != "wait":
        return True
    v = me.waited + 1
    if v > a[1]:
        return True
    return all(me.flags[f][v % 3] == 1 for f in range(len(me.nbrs)))


def last_write_before(rank, buf, e):
    w = [i for i, (_, wb) in rank.ops.items() if wb == buf and i < e]
    return max(w) if w else None


def execute(ranks, me, log):
    a = me.actions[0]
    kind = a[0]
    if kind == "wait":
        v = me.waited + 1
        if v > a[1]:
            me.actions.pop(0)
            return
        for f in range(len(me.nbrs)):             # consume slot v % 3 of every face
            assert me.flags[f][v % 3] == 1
            me.flags[f][v % 3] = 0
        me.waited = v
        log.append((me.r, "consume", v))
        return
    me.actions.pop(0)
    e = a[1]
    if kind == "read":
        # the ghosts must hold the neighbours' most recent write of that buffer before
        # operation e (all ranks run the same program)
        buf = me.ops[e][0]
        want = last_write_before(me, buf, e)
        for f in range(len(me.nbrs)):
            assert me.ghost[f][buf] == want, (me.r, e, f, buf, me.ghost[f][buf], want)
        me.reads_done.add(e)
    elif kind == "write":
        buf = me.ops[e][1]
        for f, n in enumerate(me.nbrs):
            nb = ranks[n]
            fo = f ^ 1
            # every earlier read of this buffer by the neighbour has finished, and its
            # operation e does not read what my operation e writes
            for i, (rb, _) in nb.ops.items():
                if rb == buf and i < e:
                    assert i in nb.reads_done, (me.r, e, n, i)
            assert nb.ops[e][0] != buf
            nb.ghost[fo][buf] = e
    elif kind == "signal":
        me.epoch += 1
        assert me.epoch == e
        for f, n in enumerate(me.nbrs):
            nb = ranks[n]
            fo = f ^ 1
            assert nb.flags[fo][e % 3] == 0, ("unconsumed slot overwritten", me.r, e)
            nb.flags[fo][e % 3] = 1
        log.append((me.r, "signal", e))


def run(R, calls, seed):
    rng = random.Random(seed)
    ranks = [Rank(r, [(r - 1) % R, (r + 1) % R]) for r in range(R)]
    for rk in ranks:
        build_program(rk, calls)
    log = []
    while any(rk.actions for rk in ranks):
        ready = [rk for rk in ranks if rk.actions and enabled(ranks, rk)]
        assert ready, "deadlock"
        execute(ranks, rng.choice(ready), log)
    return ranks, log


PROGRAMS = [
    ["exchange"] + ["step"] * 6,
    ["rhs", "exchange"] + ["step"] * 4,
    ["exchange", "step", "step", "rhs", "step", "exchange", "step", "step"],
]


@pytest.mark.parametrize("R", [2, 3, 4])
@pytest.mark.parametrize("prog", range(len(PROGRAMS)))
def test_protocol_random_interleavings(R, prog):
    for seed in range(300):
        ranks, _ = run(R, PROGRAMS[prog], seed + 1000 * R)
        for rk in ranks:
            assert rk.epoch == ranks[0].epoch and rk.waited <= rk.epoch
            assert all(v == 0 or v == 1 for fl in rk.flags for v in fl)


def test_steps_repeat_the_same_flag_operations():
    """Once a step starts one consumed operation behind (epoch - waited == 1, the state a
    step leaves), every step consumes and signals the same slots: the captured graph's
    memory operations are valid for every replay (mfc_rk3_steps)."""
    ranks, log = run(3, ["exchange", "step", "step", "step", "step"], 7)
    per_step = {}
    for r, kind, v in log:
        if v >= 2:                                # operations of the steps after the first
            step = (v - 2) // 3
            per_step.setdefault((r, step), []).append((kind, v % 3))
    for r in range(3):
        seqs = [sorted(per_step[(r, k)]) for k in range(1, 3)]
        assert seqs[0] == seqs[1]
