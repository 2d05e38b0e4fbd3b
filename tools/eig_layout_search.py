"""Offline search of the eig16 shared-memory layout and half-lane -> block order (csrc/eig16.cu
kSwz / kHalfOrder) under the quarter-warp model of 16-byte shared-memory accesses: a quarter-warp
(8 lanes) costs, per instruction, the largest number of distinct addresses that share one 16-byte
bank group (address mod 8 in 16-byte units).  Counted: the block loads (4) and permuted stores (4)
of both block slots per round plus the zeroed-pair store.  Layout: the strict upper triangle of
the 16 x 16 matrix folded into 8 rows of 16 (row r holds matrix rows r and 15 - r), position XOR
kSwz[r].  Constraint of the pipelined kernel: the 8 "pilot" blocks (those holding a next-round
pair element) sit in block slot 0 of distinct lanes.
python tools/eig_layout_search.py [iters]"""
import random
import sys

N, NP = 16, 8


def aidx(i, j, sw):
    assert i < j
    if i < N // 2:
        r, pos = i, j - i - 1
    else:
        r, pos = N - 1 - i, j - 1
    return r * N + (pos ^ sw[r])


def cat_next(s):
    return 0 if s == 0 else (2 if s == 1 else (N - 1 if s == N - 2 else (s - 2 if s & 1 else s + 2)))


blocks = [(r, s) for r in range(NP) for s in range(r + 1, NP)]
pinv = {cat_next(s): s for s in range(N)}
pilot = []
for k in range(NP):
    p, q = pinv[2 * k], pinv[2 * k + 1]
    a, b = min(p, q), max(p, q)
    pilot.append(blocks.index((a // 2, b // 2)))


def accesses(t, sw):
    r, s = blocks[t]
    i0, i1, j0, j1 = 2 * r, 2 * r + 1, 2 * s, 2 * s + 1
    rd = [aidx(i0, j0, sw), aidx(i0, j1, sw), aidx(i1, j0, sw), aidx(i1, j1, sw)]
    wr = []
    for x in (cat_next(i0), cat_next(i1)):
        for y in (cat_next(j0), cat_next(j1)):
            wr.append(aidx(min(x, y), max(x, y), sw))
    return rd + wr


def wavefronts(order, sw):
    tot = 0
    for u, lanes in ((0, range(16)), (1, range(12))):
        acc = [accesses(order[16 * u + l], sw) if 16 * u + l < 28 else None for l in range(16)]
        for ins in range(8):
            for q in (range(0, 8), range(8, 16)):
                groups = {}
                for l in q:
                    if l in lanes and acc[l] is not None:
                        a = acc[l][ins]
                        groups.setdefault(a % 8, set()).add(a)
                tot += max((len(v) for v in groups.values()), default=0)
    groups = {}
    for k in range(NP):
        x, y = cat_next(2 * k), cat_next(2 * k + 1)
        a = aidx(min(x, y), max(x, y), sw)
        groups.setdefault(a % 8, set()).add(a)
    tot += max(len(v) for v in groups.values())
    return tot


def valid(order):
    return all(order.index(t) < 16 for t in pilot)


def search(iters, seed=1):
    rng = random.Random(seed)
    order = pilot + [t for t in range(28) if t not in pilot]
    sw = [0] * NP
    best = cur = wavefronts(order, sw)
    best_o, best_s = order[:], sw[:]
    T = 3.0
    for it in range(iters):
        if rng.random() < 0.3:
            r = rng.randrange(NP)
            old = sw[r]
            sw[r] = rng.randrange(N)
            w = wavefronts(order, sw)
            if w <= cur or rng.random() < pow(2.718, (cur - w) / T):
                cur = w
            else:
                sw[r] = old
        else:
            a, b = rng.randrange(28), rng.randrange(28)
            order[a], order[b] = order[b], order[a]
            if not valid(order):
                order[a], order[b] = order[b], order[a]
                continue
            w = wavefronts(order, sw)
            if w <= cur or rng.random() < pow(2.718, (cur - w) / T):
                cur = w
            else:
                order[a], order[b] = order[b], order[a]
        if cur < best:
            best, best_o, best_s = cur, order[:], sw[:]
        T = max(0.05, T * 0.9997)
    return best, best_o, best_s


if __name__ == "__main__":
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
    print("pilot blocks", pilot)
    res = min(search(iters, s) for s in range(8))
    print("wavefronts per round (lower bound 33):", res[0])
    print("kHalfOrder", res[1])
    print("kSwz", res[2])
