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
