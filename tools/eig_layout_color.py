"""Conflict-free shared-memory layout for eig16h_kernel<16> (csrc/eig16.cu), by bipartite edge colouring.

Model (ncu, profiles/README.md round 2): a 16-byte shared-memory access (LDS/STS.128) is served per
quarter-warp (8 lanes); it takes one wavefront when the 8 addresses fall in 8 distinct 16-byte bank
groups (address/16 mod 8), more otherwise.  Per round every off-diagonal element (i < j) of the
slot-ordered 16 x 16 matrix is read by exactly one (instruction, quarter) group — a block load of
pass 1 / pass 2 or phase 1's pair-element load — and written by exactly one group: the permuted
store of the lane that rotated it (the caterpillar slot permutation pi) or phase 1's zeroed pair
element.  Colour every element with its bank group: each load group and each store group must be
rainbow.  That is a proper edge colouring of the bipartite multigraph (load groups) x (store
groups) with one edge per element and degree <= 8, which exists with 8 colours (Konig); this
script finds one with alternating-path (Kempe) recolouring and emits the tables.

Lane -> block assignment (pass 1: 16 blocks, pass 2: 12): the 28 off-diagonal 2x2 blocks (r < s of
8 slot pairs) are grouped by their row pair r into 12 pairs of blocks (r, s_a), (r, s_b) plus 4
singles, so a lane's pass-2 block shares the row pair with its pass-1 block and reuses its
rotation parameters (pass 2 loads one pair's parameters instead of two).

    python tools/eig_layout_color.py > /tmp/tables.txt      (paste into csrc/eig16.cu)
"""
import sys

N, NP = 16, 8


def cat_next(s):
    return 0 if s == 0 else (2 if s == 1 else (N - 1 if s == N - 2 else (s - 2 if s & 1 else s + 2)))


def blocks_assignment():
    singles, pairs = [], []
    for r in range(NP - 1):
        ss = list(range(r + 1, NP))
        while len(ss) >= 2:
            pairs.append(((r, ss.pop(0)), (r, ss.pop(0))))
        singles += [(r, s) for s in ss]
    assert len(pairs) == 12 and len(singles) == 4
    lanes = [(a, b) for a, b in pairs] + [(s, None) for s in singles]   # lane -> (pass1, pass2)
    return lanes


def elems(blk):
    r, s = blk
    return [(2 * r, 2 * s), (2 * r, 2 * s + 1), (2 * r + 1, 2 * s), (2 * r + 1, 2 * s + 1)]


def perm_pos(i, j):
    x, y = cat_next(i), cat_next(j)
    return (x, y) if x < y else (y, x)


def main():
    lanes = blocks_assignment()
    load_group, store_group = {}, {}
    groups = 0
    # pass 1 (lanes 0-15) and pass 2 (lanes 0-11): instruction e, quarter q
    for u in range(2):
        for e in range(4):
            for q in range(2):
                gid_l = ("L", u, e, q)
                gid_s = ("S", u, e, q)
                for l in range(8 * q, 8 * q + 8):
                    blk = lanes[l][u]
                    if blk is None:
                        continue
                    p = elems(blk)[e]
                    load_group[p] = gid_l
                    store_group[perm_pos(*p)] = gid_s
    for k in range(NP):                                  # phase 1: lanes 0-7 (quarter 0)
        p = (2 * k, 2 * k + 1)
        load_group[p] = ("L", "ph1")
        store_group[perm_pos(*p)] = ("S", "ph1")
    pos = [(i, j) for i in range(N) for j in range(i + 1, N)]
    assert set(load_group) == set(pos) and set(store_group) == set(pos)
    # bipartite edge colouring, Kempe chains
    C = 8
    at = {}                                              # node -> {colour: position}
    col = {}

    def free(node):
        used = at.setdefault(node, {})
        return [c for c in range(C) if c not in used]

    for p in pos:
        u, v = load_group[p], store_group[p]
        fu, fv = free(u), free(v)
        common = [c for c in fu if c in fv]
        if common:
            c = common[0]
        else:
            a, b = fu[0], fv[0]                          # a free at u, b free at v; flip the a/b path from v
            path, node, cc = [], v, a
            while cc in at.setdefault(node, {}):
                q = at[node][cc]
                path.append(q)
                other = store_group[q] if load_group[q] == node else load_group[q]
                node, cc = other, (b if cc == a else a)
            for q in path:                               # remove, then re-add with swapped colours
                at[load_group[q]].pop(col[q]); at[store_group[q]].pop(col[q])
            for q in path:
                col[q] = b if col[q] == a else a
                at[load_group[q]][col[q]] = q; at[store_group[q]][col[q]] = q
            c = a
        col[p] = c
        at[u][c] = p
        at[v][c] = p
    # verify rainbow groups
    for gmap in (load_group, store_group):
        seen = {}
        for p, g in gmap.items():
            key = (g, col[p])
            assert key not in seen, ("conflict", g, p, seen[key])
            seen[key] = p
    # physical slots: colour c -> c, c + 8, c + 16, ...
    cnt = [0] * C
    slot = {}
    for p in pos:
        c = col[p]
        slot[p] = c + 8 * cnt[c]
        cnt[c] += 1
    assert max(slot.values()) < 136 and len(set(slot.values())) == len(pos)
    print(f"// colour counts {cnt}; max slot {max(slot.values())}", file=sys.stderr)
    tab = [[-1] * N for _ in range(N)]
    for (i, j), sl in slot.items():
        tab[i][j] = sl
    print("__device__ constexpr unsigned char kOff16[16][16] = {")
    for i in range(N):
        print("    {" + ", ".join(str(v if v >= 0 else 255) for v in tab[i]) + "},")
    print("};")
    l1 = [blocks_index(b) for b, _ in lanes]
    l2 = [blocks_index(b) if b is not None else -1 for _, b in lanes]
    print("__device__ constexpr signed char kLaneBlk16[2][16] = {")
    print("    {" + ", ".join(map(str, l1)) + "},")
    print("    {" + ", ".join(map(str, l2)) + "}};")


def blocks_index(b):
    blocks = [(r, s) for r in range(NP) for s in range(r + 1, NP)]
    return blocks.index(b)


if __name__ == "__main__":
    main()
