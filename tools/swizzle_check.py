"""Shared-memory bank-conflict check for the CTA NTT pass layouts (dev tool).

Models csrc/ntt.cuh: in pass (s, r) thread t holds E/G groups
g = gg*T + sigma(t) of G = 2^r elements idx = B*(N>>s) + o + j*S with
S = N >> (s+r), o = g % S, B = g // S.  sigma rotates the low 6 thread bits
in the last pass (LOGN >= 10).  Shared address = sum of per-bit weights of idx
(additive padding, so address = thread base + compile-time offset).
"""

def cfg(logn):
    loge = 4 if logn >= 9 else (logn - 5 if logn >= 6 else 1)
    E = 1 << loge; N = 1 << logn; T = N // E
    npass = (logn + loge - 1) // loge
    first = logn - (npass - 1) * loge
    passes = [(0, first)] + [(first + (k - 1) * loge, loge) for k in range(1, npass)]
    return N, T, E, passes

def sigma(logn, last, t):
    if logn == 12 and last:   # five-bit rotation: the last exchange stays inside the warp
        return ((t & 15) << 1) | ((t >> 4) & 1) | (t & ~31)
    if logn >= 10 and last:
        return ((t & 31) << 1) | ((t >> 5) & 1) | (t & ~63)
    return t

def pass_idx(logn, N, T, E, s, r, last, t, k):
    G = 1 << r; S = N >> (s + r)
    gg, j = divmod(k, G)
    g = gg * T + sigma(logn, last, t)
    o = g % S; B = g // S
    return B * (N >> s) + o + j * S

W32 = [1, 2, 4, 8, 16, 33, 66, 132, 272, 552, 1088, 2176, 4352, 8704]
W64 = [1, 2, 4, 8, 16, 33, 66, 132, 264, 528, 1056, 2112, 4224, 8448]

def weights(logn, word):
    if logn < 10:
        return [1 << b for b in range(logn)]
    return (W32 if word == 4 else W64)[:logn]

def phys(idx, w):
    return sum(wb for b, wb in enumerate(w) if (idx >> b) & 1)

def degree(addrs, word):
    groups, nb = ([addrs], 32) if word == 4 else ([addrs[:16], addrs[16:]], 16)
    worst = 1
    for grp in groups:
        if not grp:
            continue
        banks = {}
        for a in set(grp):
            banks.setdefault(a % nb, set()).add(a)
        worst = max(worst, max(len(v) for v in banks.values()))
    return worst

if __name__ == "__main__":
    for logn in range(2, 14):
        N, T, E, passes = cfg(logn)
        for word in (4, 8):
            w = weights(logn, word)
            assert len({phys(i, w) for i in range(N)}) == N
            out = []
            for p, (s, r) in enumerate(passes):
                last = p == len(passes) - 1
                # bijectivity of the thread/slot map
                seen = {pass_idx(logn, N, T, E, s, r, last, t, k) for t in range(T) for k in range(E)}
                assert seen == set(range(N)), (logn, p)
                deg = 0
                for warp in range(max(1, T // 32)):
                    for k in range(E):
                        lanes = range(warp * 32, min(T, warp * 32 + 32))
                        addrs = [phys(pass_idx(logn, N, T, E, s, r, last, t, k), w) for t in lanes]
                        deg = max(deg, degree(addrs, word))
                out.append(deg)
            size = phys(N - 1, w) + 1
            print(f"logn={logn:2d} word={word} T={T:4d} passes={passes} conflict={out} smem_words={size}")

    # Vectorised exchange maps of ntt.cuh (32-bit words, N = 4096): map 1 between passes 0 and 1
    # (pass 0 side 64-bit), map 2 between passes 1 and 2 (pass 2 side 128-bit).  Vector accesses
    # are modelled per phase (16 lanes x 8 B, 8 lanes x 16 B) and must be contiguous and aligned.
    MAPS = {1: [2, 4, 8, 16, 32, 64, 128, 256, 1, 512, 1024, 2048],
            2: [1, 2, 4, 8, 16, 36, 72, 144, 304, 588, 1176, 2352]}
    logn = 12
    N, T, E, passes = cfg(logn)

    def vec_degree(w, p, vec):
        s, r = passes[p]
        last = p == len(passes) - 1
        phase = {1: 32, 2: 16, 4: 8}[vec]
        worst = 1
        for warp in range(T // 32):
            for k0 in range(0, E, vec):
                per_lane = []
                for lane in range(32):
                    ad = [phys(pass_idx(logn, N, T, E, s, r, last, warp * 32 + lane, k), w) for k in range(k0, k0 + vec)]
                    assert ad == list(range(ad[0], ad[0] + vec)) and ad[0] % vec == 0, (p, lane, k0, ad)
                    per_lane.append(ad)
                for p0 in range(0, 32, phase):
                    banks = {}
                    for ad in per_lane[p0:p0 + phase]:
                        for a in ad:
                            banks.setdefault(a % 32, set()).add(a)
                    worst = max(worst, max(len(v) for v in banks.values()))
        return worst

    for m, w in MAPS.items():
        if m == 2:
            continue  # replaced by the warp-local exchange below (kept for reference)
        assert len({phys(i, w) for i in range(N)}) == N
        sides = [(0, 2), (1, 1)]
        degs = [vec_degree(w, p, v) for p, v in sides]
        assert degs == [1, 1], (m, degs)
        print(f"vector map {m}: sides (pass, words) {sides} conflict={degs} smem_words={phys(N - 1, w) + 1}")

    # map 1 keeps index bits 9-11 as address bits 9-11: the middle pass touches only its warp's block
    w1 = MAPS[1]
    s1, r1 = passes[1]
    for t in range(T):
        for k in range(E):
            assert phys(pass_idx(logn, N, T, E, s1, r1, False, t, k), w1) // 512 == t // 32
    # and the first-pass side is thread-stationary (forward's writes == inverse's reads): same layout

    # Warp-local exchange between the middle and the last pass (ntt.cuh Exchanger::run_warp): both
    # sides must address every element identically, inside the warp's 512-word block, conflict-free.
    def mid_addr(t, m):
        mid = 272 * ((t >> 4) & 1) + (t & 15)
        return (t & ~31) * 16 + ((mid ^ (4 * (m >> 1))) + 32 * (m & 7))

    def last_addr(t, k):
        sl = (t >> 3) & 1
        row = 256 * sl + 32 * (((t & 3) << 1) | ((t >> 4) & 1)) + 16 * (((t >> 2) & 1) ^ sl) + 4 * (t & 3)
        return (t & ~31) * 16 + (row ^ (4 * (k // 4))) + (k % 4)

    s2, r2 = passes[2]
    where = {}
    for t in range(T):
        for k in range(E):
            a = mid_addr(t, k)
            assert a // 512 == t // 32
            idx = pass_idx(logn, N, T, E, s1, r1, False, t, k)
            assert idx not in where
            where[idx] = a
    assert len(set(where.values())) == N
    for t in range(T):
        for k in range(E):
            assert where[pass_idx(logn, N, T, E, s2, r2, True, t, k)] == last_addr(t, k), (t, k)
    worst_s = worst_v = 1
    for warp in range(T // 32):
        for k in range(E):
            worst_s = max(worst_s, degree([mid_addr(warp * 32 + l, k) for l in range(32)], 4))
        for c in range(4):
            for q in range(4):
                banks = {}
                for l in range(8 * q, 8 * q + 8):
                    for i in range(4):
                        a = last_addr(warp * 32 + l, 4 * c + i)
                        banks.setdefault(a % 32, set()).add(a)
                worst_v = max(worst_v, max(len(v) for v in banks.values()))
    assert (worst_s, worst_v) == (1, 1), (worst_s, worst_v)
    print(f"warp-local exchange (passes 1 <-> 2): both sides agree, inside the warp's block, conflict={[worst_s, worst_v]}")
