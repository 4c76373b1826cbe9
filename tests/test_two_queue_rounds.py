"""Host model of the codebook kernel's batched two-queue merge
(csrc/codebook.cu: two_queue) against the sequential merge it must reproduce
(the reference's K.huffman_lengths, _kernels.py:213-232: two FIFO queues,
the leaf wins ties).  The GPU tests compare the kernel with the oracle; this
pins the ALGORITHM -- every round rule, the carry, the empty-queue case --
on weight sets chosen to stress ties and growth, without a GPU."""
import bisect

import numpy as np
import pytest


def sequential(L):
    k = len(L)
    inf = 1 << 62
    W = [0] * (k - 1)
    PL = [0] * k
    PI = [0] * (k - 1)
    leaf = node = 0
    for nI in range(k - 1):
        s = 0
        for _ in range(2):
            wl = L[leaf] if leaf < k else inf
            wi = W[node] if node < nI else inf
            if wl <= wi:  # leaf wins ties
                s += wl
                PL[leaf] = nI
                leaf += 1
            else:
                s += wi
                PI[node] = nI
                node += 1
        W[nI] = s
    return PL, PI


def batched(L):
    """Mirror of two_queue(): one round settles every pick up to the last
    existing node; ranks by binary search; odd last pick carried."""
    k = len(L)
    Iw = [0] * k
    PL = [0] * k
    PI = [0] * k
    leaf = node = nI = 0
    carry = 0
    cidx = cw = 0
    rounds = 0
    while nI < k - 1:
        rounds += 1
        e = nI - node
        if e == 0:
            s = 0
            lf = leaf
            if carry == 1:
                PL[cidx] = nI
                s += cw
            elif carry == 2:
                PI[cidx] = nI
                s += cw
            for _ in range(1 if carry else 0, 2):
                s += L[lf]
                PL[lf] = nI
                lf += 1
            Iw[nI] = s
            leaf = lf
            nI += 1
            carry = 0
            continue
        wmax = Iw[nI - 1]
        cL = bisect.bisect_right(L, wmax, leaf, k) - leaf
        T = cL + e
        c = 1 if carry else 0
        odd = (T + c) & 1
        if carry:
            if carry == 1:
                PL[cidx] = nI
            else:
                PI[cidx] = nI
            Iw[nI] += cw
        ncarry = -1
        for t in range(T):
            if t < cL:
                w = L[leaf + t]
                pos = t + (bisect.bisect_left(Iw, w, node, node + e) - node) + c
                PL[leaf + t] = nI + (pos >> 1)
                Iw[nI + (pos >> 1)] += w
            else:
                j = t - cL
                w = Iw[node + j]
                pos = j + (bisect.bisect_right(L, w, leaf, leaf + cL) - leaf) + c
                if odd and pos == T + c - 1:
                    ncarry = node + j
                else:
                    PI[node + j] = nI + (pos >> 1)
                    Iw[nI + (pos >> 1)] += w
        leaf += cL
        node = nI
        nI += (T + c) >> 1
        if odd:
            carry, cidx, cw = 2, ncarry, Iw[ncarry]
        else:
            carry = 0
    return PL, PI[:k - 1], rounds


def _weights(kind, k, rng):
    if kind == "small-ints":
        return rng.integers(1, 5, k)
    if kind == "wide":
        return rng.integers(1, 1 << 20, k)
    if kind == "ones":
        return np.ones(k, np.int64)
    if kind == "bell":
        return (np.exp(-np.linspace(-4, 4, k) ** 2) * 1e6).astype(np.int64) + 1
    if kind == "geometric-growth":
        return np.array([int(1.3 ** i) + 1 for i in range(min(k, 60))])
    return rng.geometric(0.01, k)


@pytest.mark.parametrize("kind", ["small-ints", "wide", "ones", "bell", "geometric-growth",
                                  "geometric-dist"])
def test_batched_rounds_equal_sequential_merge(kind):
    rng = np.random.default_rng(hash(kind) % 1000)
    worst = 0
    for k in [2, 3, 4, 5, 7, 8, 33, 100, 257, 1000, int(rng.integers(2, 1500))]:
        L = sorted(int(x) for x in _weights(kind, k, rng))
        a = sequential(L)
        b = batched(L)
        n = len(L)
        assert a[0] == b[0], (kind, n, "leaf parents")
        assert a[1][:n - 2] == b[1][:n - 2], (kind, n, "node parents")
        worst = max(worst, b[2])
    # every live node is consumed in the round after its creation: the rounds
    # follow the tree height, not k
    assert worst <= 130


def test_round_count_is_height_bound_for_a_large_bell():
    k = 20000
    w = (np.exp(-np.linspace(-4.5, 4.5, k) ** 2 / 2) * 3e3).astype(np.int64) + 1
    L = sorted(int(x) for x in w)
    a = sequential(L)
    b = batched(L)
    assert a[0] == b[0] and a[1][:k - 2] == b[1][:k - 2]
    assert b[2] <= 64
