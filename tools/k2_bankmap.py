"""Line -> lane map and accumulator padding for K2's line phase that minimise
shared-memory bank conflicts (dev tool; its output is pasted into
csrc/kernel_residual_map.cuh).

K2's line phase is bound by the shared-memory data pipe (ncu: l1tex data-pipe
wavefronts at 93% of peak, 1.65 wavefronts per ideal one): every 64-bit access
of a half-warp (16 lanes) costs as many wavefronts as the worst bank pair is
hit, the bank pair being the double index mod 16. A lane's double index is
    base(region, b) + doff(region, dir) + L(dir, line) + a * stride(dir)
with PRIM/COF bases fixed by the TMA block layout and the accumulator strides
free (padding). All lanes of a warp run the same (region, a) access at the same
time, so the cost of a map is sum over half-warps and (region, a) of
weight(region, a) * max multiplicity of the residues.

    python tools/k2_bankmap.py N [seconds]
"""
import math
import random
import sys
import time

N = int(sys.argv[1]) if len(sys.argv) > 1 else 5
SECS = float(sys.argv[2]) if len(sys.argv) > 2 else 60
N2, N3 = N * N, N * N * N
LINES = 3 * N2
EPB = 6 if LINES <= 32 else (4 if LINES <= 64 else (1 if N >= 6 else 2))
THREADS = ((EPB * LINES + 31) // 32) * 32
NHW = THREADS // 16
# accesses per line by (region, a): PRIM 6 arrays, COF 3, ACC 10 (5 loads + 5 stores)
asb = list(range(N))                                 # as node b in the volume pairs: b times
asa = [1] * (N - 1) + [0]                            # as node a
W = {"P": [6 * (asa[a] + asb[a] + 2) for a in range(N)],
     "C": [3 * (asa[a] + asb[a] + 2 + 2) for a in range(N)],
     "A": [10 * (asb[a] + asa[a] + 2) for a in range(N)]}
STRIDE = (1, N, N2)


def lbase(d, t1, t2):
    return N * (t1 + N * t2) if d == 0 else (t1 + N2 * t2 if d == 1 else t1 + N * t2)


lines = [(b, d, t1, t2) for b in range(EPB) for d in range(3) for t2 in range(N) for t1 in range(N)]


def residues(line, pad):
    """per (region, a) residue of one line; pad = (ES_A, DA1, DA2) mod 16"""
    b, d, t1, t2 = line
    lb = lbase(d, t1, t2)
    esa, da1, da2 = pad
    da = (0, da1, da2)[d]
    out = []
    for a in range(N):
        o = lb + a * STRIDE[d]
        out.append(((6 * N3 * b + o) % 16, (9 * N3 * b + N3 * d + o) % 16, (esa * b + da + o) % 16))
    return out


def hw_cost(members, pad, cache):
    c = 0
    for a in range(N):
        cnt = ([0] * 16, [0] * 16, [0] * 16)
        for ln in members:
            if ln is None:
                continue
            r = cache[ln][a]
            cnt[0][r[0]] += 1
            cnt[1][r[1]] += 1
            cnt[2][r[2]] += 1
        c += W["P"][a] * max(cnt[0]) + W["C"][a] * max(cnt[1]) + W["A"][a] * max(cnt[2])
    return c


def ideal():
    # one wavefront per access of a non-empty half-warp, EPB*LINES lanes packed
    full = math.ceil(EPB * LINES / 16)
    return full * sum(sum(v) for v in W.values())


def total(slots, pad, cache):
    return sum(hw_cost(slots[16 * h:16 * h + 16], pad, cache) for h in range(NHW))


def natural():
    s = [None] * THREADS
    for t in range(EPB * LINES):
        b, ll = divmod(t, LINES)
        d, lrem = divmod(ll, N2)
        s[t] = lines.index((b, d, lrem % N, lrem // N))
    return s


def anneal(pad, secs, seed):
    rng = random.Random(seed)
    cache = [residues(l, pad) for l in lines]
    slots = natural()
    cost = [hw_cost(slots[16 * h:16 * h + 16], pad, cache) for h in range(NHW)]
    cur = sum(cost)
    best, best_slots = cur, slots[:]
    t0, T = time.time(), 30.0
    it = 0
    while time.time() - t0 < secs:
        it += 1
        if it % 2000 == 0:
            T = max(0.05, 30.0 * (1 - (time.time() - t0) / secs) ** 2)
        i, j = rng.randrange(THREADS), rng.randrange(THREADS)
        hi, hj = i // 16, j // 16
        if hi == hj or (slots[i] is None and slots[j] is None):
            continue
        slots[i], slots[j] = slots[j], slots[i]
        ci = hw_cost(slots[16 * hi:16 * hi + 16], pad, cache)
        cj = hw_cost(slots[16 * hj:16 * hj + 16], pad, cache)
        d = ci + cj - cost[hi] - cost[hj]
        if d <= 0 or rng.random() < math.exp(-d / T):
            cost[hi], cost[hj] = ci, cj
            cur += d
            if cur < best:
                best, best_slots = cur, slots[:]
        else:
            slots[i], slots[j] = slots[j], slots[i]
    return best, best_slots


if __name__ == "__main__":
    pad0 = ((15 * N3) % 16, (5 * N3) % 16, (10 * N3) % 16)
    cache0 = [residues(l, pad0) for l in lines]
    nat = total(natural(), pad0, cache0)
    print(f"N={N} EPB={EPB} threads={THREADS}: ideal {ideal()}, natural map {nat} ({nat / ideal():.3f}x)")
    best = None
    rng = random.Random(1)
    cands = [pad0] + [(rng.randrange(16), rng.randrange(16), rng.randrange(16)) for _ in range(11)]
    for k, pad in enumerate(cands):
        c, s = anneal(pad, SECS / len(cands), k)
        print(f"  pad (ES_A, DA1, DA2) mod 16 = {pad}: {c} ({c / ideal():.3f}x)", flush=True)
        if best is None or c < best[0]:
            best = (c, s, pad)
    c, s, pad = best
    print(f"best {c} ({c / ideal():.3f}x) with pad {pad}")
    codes = []
    for t in range(THREADS):
        if s[t] is None:
            codes.append(0xFFFF)
        else:
            b, d, t1, t2 = lines[s[t]]
            codes.append(b << 12 | d << 8 | t2 << 4 | t1)
    print("map:", ", ".join(f"0x{x:04x}" for x in codes))
