"""N1 NCCL baseline (ADAPTRA_EXEC_NCCL, csrc/exec/exec.cpp run_nccl): its issue
pattern checked on CPU for every arm's per-stage orders.  Per op, the
executor groups the previous op's send with this op's receive
(ncclGroupStart/End); NCCL matches point-to-point operations between two
ranks in issue order and a group -- one kernel on the stage's stream --
completes only when all of its operations have.  So (1) on every link and
direction the sends must carry the microbatches in the order the receiver
posts its receives (else data would land in the wrong mailbox slot), and (2)
the groups must never deadlock.  A discrete simulation of the blocking
groups checks both.  Its model: a send completes once its receive is posted,
or on its own while fewer than K earlier messages of its link sit unreceived
in NCCL's buffers (K = 0: strict rendezvous; K = None: unbounded); a receive
completes once posted and its send has completed.

Finding (DESIGN R39): with each receive posted alongside its own op, 1F1B
never deadlocks even at K = 0, but orders with many warm-up forwards (Alg.
2's adapted orders, the greedy ZB orders) need K of several messages --
stage 0 blocked sending F_k while stage 1 is blocked sending B_1.  The
paper's adaptation assumes this away: "we assume no HOL blocking stalls --
which is guaranteed by our second design" (Sec. 5 intro).
The executor therefore takes a receive-posting plan (adaptra_nccl_post_plan,
given the K the binding measures on the live communicator) that hoists a
receive into the receiver's current group only where K does not absorb the
orders; the simulator checks that plan from the outside."""
import pytest
from hypothesis import given, settings, strategies as st

import synthetic as sy
from paper_2504_19232_b200 import _lib as L, sched as cs
from paper_2504_19232_b200.pipeline import Arm


def recv_of(k, i, S):
    if k == "F" and i > 0:
        return (i - 1, "f")
    if k == "B" and i < S - 1:
        return (i + 1, "b")
    return None


def send_of(k, i, S):
    if k == "F" and i < S - 1:
        return (i + 1, "f")
    if k == "B" and i > 0:
        return (i - 1, "b")
    return None


def groups(order, i, S, merge, post=None):
    """The executor's NCCL groups of stage i: [(sends, recvs)], each a list
    of (peer, direction, mb).  Group p goes before op p's kernels and holds
    op p-1's send and the receives of the ops q with post[q] == p (default
    q: each receive with its own op)."""
    n = len(order)
    if post is None:
        post = [q if recv_of(k, i, S) else -1 for q, (k, _) in enumerate(order)]
    out = []
    for p in range(n + 1):
        snd = []
        if p > 0 and send_of(order[p - 1][0], i, S):
            snd = [send_of(order[p - 1][0], i, S) + (order[p - 1][1],)]
        rcv = [recv_of(order[q][0], i, S) + (order[q][1],) for q in range(p, n) if post[q] == p]
        if snd or rcv:
            out.append((snd, rcv))
    return out


def simulate(orders, S, merge, buffered=0, post=None):
    G = [groups(orders[i], i, S, merge, post[i] if post else None) for i in range(S)]
    # (1) per channel (src, dst, dir) the sends carry the microbatches in the
    # order the receiver posts its receives
    sent, recvd, where = {}, {}, {}
    for i in range(S):
        for gi, (snd, rcv) in enumerate(G[i]):
            for (j, d, mb) in snd:
                ch = (i, j, d)
                where[(ch, len(sent.setdefault(ch, [])), "s")] = (i, gi)
                sent[ch].append(mb)
            for (j, d, mb) in rcv:
                ch = (j, i, d)
                where[(ch, len(recvd.setdefault(ch, [])), "r")] = (i, gi)
                recvd[ch].append(mb)
    assert sent == recvd, "send and receive orders differ on a link"
    # (2) the blocking groups, operation by operation
    members = [[[] for _ in G[i]] for i in range(S)]
    for key, (i, gi) in where.items():
        members[i][gi].append(key)
    done = set()
    pos = [0] * S

    def is_posted(key):
        i, gi = where[key]
        return pos[i] == gi

    def unreceived(ch, k):   # messages before k on ch sent but not yet received
        return sum(1 for kk in range(k) if (ch, kk, "s") in done and (ch, kk, "r") not in done)

    while any(pos[i] < len(G[i]) for i in range(S)):
        progress = False
        for i in range(S):
            if pos[i] >= len(G[i]):
                continue
            for key in members[i][pos[i]]:
                if key in done:
                    continue
                ch, k, role = key
                if role == "s":
                    r = (ch, k, "r")
                    if is_posted(r) and all((ch, kk, "r") in done for kk in range(k)):
                        done.add(key)                      # matched
                        progress = True
                    elif buffered is None or unreceived(ch, k) < buffered:
                        done.add(key)                      # absorbed by the buffers
                        progress = True
                elif (ch, k, "s") in done:
                    done.add(key)
                    progress = True
        for i in range(S):
            if pos[i] < len(G[i]) and all(k in done for k in members[i][pos[i]]):
                pos[i] += 1
                progress = True
        assert progress, f"NCCL deadlock at group positions {pos}"


def hoisted(orders, post, S):
    return sum(1 for i in range(S) for q, (k, _) in enumerate(orders[i])
               if recv_of(k, i, S) and post[i][q] != q)


@st.composite
def cases(draw):
    S = draw(st.integers(2, 8))
    N = draw(st.integers(1, 32))
    seed = draw(st.integers(0, 10 ** 6))
    tF, tB, tW, _ = sy.stage_profile(seed, S, 1, 40)
    arm = draw(st.sampled_from(["zb", "1f1b", "adaptive"]))
    c = sy.stage_profile(seed + 1, S, 1, 2, draw(st.sampled_from([0, 30, 200])))[3]
    a = Arm(arm, S, N, tF, tB, tW)
    return a.plan(c), S, a.merge_w, arm


@settings(max_examples=200, deadline=None)
@given(cases(), st.sampled_from([0, 1, 2, 4]))
def test_nccl_issue_pattern_matches_and_never_deadlocks(case, K):
    """Every arm's orders match per channel and never deadlock with unbounded
    buffers; with the receive-posting plan for K buffered messages they never
    deadlock at K either; the plan only moves receives earlier, and not at
    all where K already absorbs the orders (the baseline is not slowed by
    needless early receives)."""
    orders, S, merge, arm = case
    simulate(orders, S, merge, buffered=None)
    post = cs.nccl_post_plan(orders, merge, K)
    for i in range(S):
        for q, (k, _) in enumerate(orders[i]):
            if recv_of(k, i, S):
                assert 0 <= post[i][q] <= q
            else:
                assert post[i][q] == -1
    simulate(orders, S, merge, buffered=K, post=post)
    try:
        simulate(orders, S, merge, buffered=K)
    except AssertionError:
        assert hoisted(orders, post, S) > 0
    else:
        assert hoisted(orders, post, S) == 0


def test_1f1b_needs_no_buffering():
    """1F1B's pairing (send_forward_recv_backward) is deadlock-free even at
    strict rendezvous, so its plan is the identity."""
    for S, N in ((2, 4), (4, 16), (8, 32)):
        t = [1000] * S
        a = Arm("1f1b", S, N, t, t, t)
        orders = a.plan([0] * (S - 1))
        simulate(orders, S, a.merge_w, buffered=0)
        assert hoisted(orders, cs.nccl_post_plan(orders, a.merge_w, 0), S) == 0


def test_adapted_orders_deadlock_without_the_receive_plan():
    """R39: the 2-stage case with a 3 ms link on N=6: Alg. 2 gives stage 0
    six warm-up forwards; with each receive posted with its own op and no
    buffering, stage 1 blocks sending B1 (stage 0 receives it only after F6)
    while stage 0 blocks sending F3 (stage 1 posts that receive only after
    its B2 send) -- a cycle.  The K = 0 plan posts stage 1's receives of
    F3..F5 in its group 2 (with the B1 send), so stage 0's warm-up forwards
    flow on; with K = 3 buffered messages nothing needs to move."""
    S, N, t = 2, 6, [1000, 1000]
    a = Arm("adaptive", S, N, t, t, t)
    orders = a.plan([3000])
    assert [k for k, _ in orders[0][:7]] == ["F"] * 6 + ["B"]
    simulate(orders, S, a.merge_w, buffered=None)
    with pytest.raises(AssertionError, match="deadlock"):
        simulate(orders, S, a.merge_w, buffered=0)
    post = cs.nccl_post_plan(orders, a.merge_w, 0)
    f = {mb: q for q, (k, mb) in enumerate(orders[1]) if k == "F"}
    assert [post[1][f[m]] for m in (3, 4, 5)] == [2, 2, 2]
    simulate(orders, S, a.merge_w, buffered=0, post=post)
    simulate(orders, S, a.merge_w, buffered=3)
    assert hoisted(orders, cs.nccl_post_plan(orders, a.merge_w, 3), S) == 0


def test_post_plan_rejects_mismatched_orders():
    crossed = [[("F", 1), ("F", 2), ("B", 2), ("B", 1)], [("F", 2), ("F", 1), ("B", 1), ("B", 2)]]
    with pytest.raises(L.AdaptraError):
        cs.nccl_post_plan(crossed)


def test_simulator_detects_a_deadlock():
    """A crossed pair of orders is reported, and so is a blocking cycle."""
    S = 2
    crossed = [[("F", 1), ("F", 2), ("B", 2), ("B", 1)], [("F", 2), ("F", 1), ("B", 1), ("B", 2)]]
    with pytest.raises(AssertionError, match="orders differ"):
        simulate(crossed, S, False)
    # stage 0 sends three forwards before its first backward, stage 1 is
    # 1F1B: the channel orders match, but with receives posted per op and
    # no buffering stage 0 blocks sending F3 while stage 1 blocks sending B1;
    # one buffered message absorbs it
    cyc = [[("F", m) for m in range(1, 5)] + [("B", m) for m in range(1, 5)],
           [(k, m) for m in range(1, 5) for k in "FB"]]
    simulate(cyc, S, True, buffered=None)
    with pytest.raises(AssertionError, match="deadlock"):
        simulate(cyc, S, True, buffered=0)
    simulate(cyc, S, True, buffered=1)
    simulate(cyc, S, True, buffered=0, post=cs.nccl_post_plan(cyc, True, 0))
