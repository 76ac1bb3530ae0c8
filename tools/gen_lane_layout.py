"""Search bank-conflict-free line-buffer layouts for the 3D warp tiles
(Q2: 3 cells x 9 lines per warp; Q4: 1 cell x 25 lines), 64-bit shared
accesses served per half-warp.

A layout = (which (cell, line) slot each lane holds, split over the two
half-warps) + a 16-colouring of the (cell, point) sites such that in every
axis phase and line position the sites one half-warp touches have distinct
colours; the address of a site is colour + 16 * (index within its colour
class).  The cache is read per slot, so each half's slots are also kept
distinct mod 16.  Emits paper_1904_13131_b200/csrc/hf_lanemap.h.

    python tools/gen_lane_layout.py
"""
import os
import random

DIM = 3
# (N, cells per warp).  (5, 1) -- 3D Q4 -- also has a conflict-free layout
# (COMP 128), but it measured no faster on B200 (+14 registers for the offsets,
# b2b 48.1 -> 48.5 us tensor4 at config 3): `python tools/gen_lane_layout.py 5`.
CASES = [(3, 3)]


def line_pts(n, ax, t, l):
    if ax == 0:
        return (l, t % n, t // n)
    if ax == 1:
        return (t % n, l, t // n)
    return (t % n, t // n, l)


def colour(n, cpw, groups, rnd, ncol=16, tries=50):
    verts = [(m, i, j, k) for m in range(cpw) for i in range(n) for j in range(n) for k in range(n)]
    nbr = {v: set() for v in verts}
    for ax in range(DIM):
        for l in range(n):
            for g in groups:
                cl = [(m,) + line_pts(n, ax, t, l) for (m, t) in g]
                for a in cl:
                    nbr[a].update(b for b in cl if b != a)
    for _ in range(tries):
        col, cnt, unc = {}, [0] * ncol, set(verts)
        while unc:
            v = max(unc, key=lambda v: (len({col[u] for u in nbr[v] if u in col}), len(nbr[v]), rnd.random()))
            free = [c for c in range(ncol) if c not in {col[u] for u in nbr[v] if u in col}]
            if not free:
                break
            c = min(free, key=lambda c: (cnt[c], rnd.random()))
            col[v] = c
            cnt[c] += 1
            unc.remove(v)
        else:
            return col
    return None


def layout(n, cpw):
    rnd = random.Random(7)
    L = n * n
    slots = [(m, t) for m in range(cpw) for t in range(L)]
    half = (len(slots) + 1) // 2
    best, target = None, -(-cpw * n ** 3 // 16)  # smallest possible colour class
    for _ in range(20000):
        perm = slots[:]
        rnd.shuffle(perm)
        groups = [perm[:half], perm[half:]]
        if any(len({(m * L + t) % 16 for m, t in g}) != len(g) for g in groups):
            continue
        col = colour(n, cpw, groups, rnd)
        if col:
            size = max(list(col.values()).count(c) for c in set(col.values()))
            if best is None or size < best[0]:
                best = (size, groups, col)
            if size == target:
                break
    if best is None:
        raise SystemExit(f"no layout found for N={n}")
    _, groups, col = best
    idx, addr = {}, {}
    for v in sorted(col):
        c = col[v]
        addr[v] = c + 16 * idx.get(c, 0)
        idx[c] = idx.get(c, 0) + 1
    comp = 16 * max(idx.values())
    lane_slot = [-1] * 32
    for h, g in enumerate(groups):
        for k, (m, t) in enumerate(g):
            lane_slot[16 * h + k] = m * L + t
    S = cpw * L
    off = [[[addr[(s // L,) + line_pts(n, ax, s % L, l)] for l in range(n)] for ax in range(DIM)] for s in range(S)]
    for ax in range(DIM):  # verify: every half-warp access hits distinct banks
        for l in range(n):
            for h in range(2):
                banks = [off[lane_slot[16 * h + k]][ax][l] % 16 for k in range(16) if lane_slot[16 * h + k] >= 0]
                assert len(banks) == len(set(banks))
    assert sorted(addr.values()) == sorted(set(addr.values())) and max(addr.values()) < comp
    return comp, lane_slot, off


def emit(f, n, comp, lane_slot, off):
    words = [0, 0, 0]
    for lane, sl in enumerate(lane_slot):
        words[lane // 12] |= (31 if sl < 0 else sl) << (5 * (lane % 12))
    f.write(f"// 3D Q{n - 1}: lanes -> slots {lane_slot}\n")
    f.write(f"template <>\nstruct LaneMapT<3, {n}> {{\n  static constexpr bool ENABLED = true;\n")
    f.write(f"  static constexpr int COMP = {comp};  // doubles per component block of a warp's line buffer\n")
    f.write("  // slot of each lane as 5-bit fields of three immediates (31 = idle): no memory access\n")
    f.write("  static constexpr unsigned long long B0 = 0x%xull, B1 = 0x%xull, B2 = 0x%xull;\n" % tuple(words))
    bits = max(1, (comp - 1).bit_length())
    per = 64 // bits
    nw = -(-3 * n // per)
    table = []
    for lane, sl in enumerate(lane_slot):
        w = [0] * nw
        if sl >= 0:
            for k, v in enumerate(off[sl][a][l] for a in range(3) for l in range(n)):
                w[k // per] |= v << (bits * (k % per))
        table.append(w)
    f.write(f"  // buffer offset of the site at position l along axis a of the lane's line: {bits}-bit\n"
            f"  // fields of a per-lane table that the launcher passes as a kernel parameter\n"
            f"  // (TabLine::loff: constant bank, no memory round trip at kernel start)\n")
    f.write(f"  static constexpr int OFF_BITS = {bits}, OFF_WORDS = {nw};\n")
    f.write(f"  static constexpr unsigned long long TABLE[32][{nw}] = {{\n")
    for lane, w in enumerate(table):
        f.write("      {" + ", ".join(f"0x{v:x}ull" for v in w) + f"}},  // lane {lane}\n")
    f.write("  };\n};\n\n")


def main():
    import sys
    cases = CASES + [(5, 1)] if "5" in sys.argv[1:] else CASES
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1904_13131_b200", "csrc",
                       "hf_lanemap.h")
    with open(out, "w") as f:
        f.write("// Generated by tools/gen_lane_layout.py: bank-conflict-free line-buffer layouts of the\n")
        f.write("// 3D warp tiles (lane -> (cell, line) slot; per-slot site offsets per axis phase).\n")
        f.write("#pragma once\nnamespace hf {\n\n")
        f.write("template <int DIM, int N>\nstruct LaneMapT {\n  static constexpr bool ENABLED = false;\n"
                "  static constexpr int COMP = 0;\n};\n\n")
        for n, cpw in cases:
            comp, lane_slot, off = layout(n, cpw)
            emit(f, n, comp, lane_slot, off)
            print(f"N={n} COMP={comp} lanes={lane_slot}")
        f.write("}  // namespace hf\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
