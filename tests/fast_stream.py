"""NumPy restatement of the FAST-mode random stream (test infrastructure).

Philox4x32-10 (Salmon et al., SC'11; Random123) and the FAST counter layout of
include/samegibbs_b200.h (SG_RNG_FAST): fixed key (FAST_K0, FAST_K1), counter
(global case, v | quad << 16 | purpose << 28, step key lo, step key hi); word
j of a block belongs to replica 4 * quad + j.  The device implementation is
csrc/sg_device.cuh (fast_key / fast_case / fast_draw).
"""

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
FAST_K0, FAST_K1 = 0x243F6A88, 0x85A308D3
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """Vectorised Philox4x32-10: ctr uint32 (..., 4), key (k0, k1) ints or arrays."""
    x = [np.asarray(ctr[..., i], dtype=np.uint64) for i in range(4)]
    k0 = np.asarray(key[0], dtype=np.uint64)
    k1 = np.asarray(key[1], dtype=np.uint64)
    for r in range(10):
        if r:
            k0 = (k0 + np.uint64(W0)) & MASK
            k1 = (k1 + np.uint64(W1)) & MASK
        p0 = np.uint64(M0) * x[0]
        p1 = np.uint64(M1) * x[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        x = [hi1 ^ x[1] ^ k0, lo1, hi0 ^ x[3] ^ k1, lo0]
    return np.stack([a.astype(np.uint32) for a in x], axis=-1)


def fast_block(key: int, gcase, v, quad, purpose):
    """FAST block(s) for step key `key` (uint64) -> uint32 (..., 4)."""
    gcase = np.asarray(gcase, dtype=np.uint64)
    word = (np.asarray(v, dtype=np.uint64) | (np.asarray(quad, dtype=np.uint64) << np.uint64(16))
            | (np.asarray(purpose, dtype=np.uint64) << np.uint64(28)))
    gcase, word = np.broadcast_arrays(gcase, word)
    ctr = np.stack([gcase & MASK, word & MASK, np.full(gcase.shape, key & 0xFFFFFFFF, dtype=np.uint64),
                    np.full(gcase.shape, key >> 32, dtype=np.uint64)], axis=-1)
    return philox4x32_10(ctr, (FAST_K0, FAST_K1))


def fast_init_states(key: int, obs: np.ndarray, cards, m: int, case_base: int = 0) -> np.ndarray:
    """Latent initial states of sg_init_states (FAST): (n, m, cases) int8 with
    the latent flag 0x80 on hidden cells; state = (word * card) >> 32."""
    n, cases = obs.shape
    out = np.zeros((n, m, cases), dtype=np.int16)
    c = np.arange(cases, dtype=np.uint64) + np.uint64(case_base)
    for v in range(n):
        for r in range(m):
            w = fast_block(key, c, v, r >> 2, 1)[:, r & 3].astype(np.uint64)
            s = ((w * np.uint64(cards[v])) >> np.uint64(32)).astype(np.int16)
            out[v, r] = np.where(obs[v] >= 0, obs[v], 0x80 | s)
    return out.astype(np.uint8).view(np.int8)


# ------------------------------------------------------------ joint sweep
# rng = "joint" (csrc/sg_small.cu, "joint sweep"): one uniform per lane drawn
# from the sweep's transition kernel K_P(S -> S'), the colour-ordered product
# of the full conditionals (reference sampler.py:217-284).

def lane_fields(cards):
    """Field widths and bit offsets of the packed lane word (netpack.small_plan)."""
    width = [max(1, (int(k) - 1).bit_length()) for k in cards]
    off = [0] * len(cards)
    for v in range(1, len(cards)):
        off[v] = off[v - 1] + width[v - 1]
    return width, off


def _conditional(onet, cpts, v, a):
    """Full conditional of v given assignment a: the weights of
    sampler.py:226-242 (parent row, then children ascending, fp64 left to
    right), sequential norm, times one reciprocal of the norm."""
    cfg = sum(int(a[p]) * st for p, st in zip(onet.parents[v], onet.strides(v)))
    w = [float(x) for x in cpts[v][cfg]]
    for c in onet.children[v]:
        cs = onet.strides(c)
        vst = cs[onet.parents[c].index(v)]
        cfg0 = sum(int(a[p]) * st for p, st in zip(onet.parents[c], cs) if p != v)
        for t in range(len(w)):
            w[t] = w[t] * float(cpts[c][cfg0 + t * vst, int(a[c])])
    norm = 0.0
    for x in w:
        norm = norm + x
    inv = 1.0 / norm if norm > 0.0 else 0.0  # one reciprocal, then products (csrc joint_conditional)
    return [x * inv for x in w]


def warp_scan(p):
    """Cumulative sums of one row in the device's order (csrc joint_slice):
    K <= 32 -- one column per lane, Kogge-Stone over the lanes; K = 64 --
    lane l holds (2l, 2l+1): its pair sum is scanned, then column 2l = the
    left neighbour's inclusive sum + p[2l], column 2l+1 = its own."""
    K = len(p)
    x = p.copy() if K <= 32 else p[0::2] + p[1::2]
    d = 1
    while d < 32:
        x[d:] = x[d:] + x[:-d]
        d *= 2
    if K <= 32:
        return x
    out = np.empty(K)
    out[1::2] = x
    out[0] = p[0]
    out[2::2] = x[:-1] + p[2::2]
    return out


def joint_tables(onet, cpts, order):
    """{P: (B, keep, dep[K], rows uint32 (R, K))} for every pattern with latent bits."""
    import math

    n = onet.n
    cards = onet.cards
    width, off = lane_fields(cards)
    bits = sum(width)
    R = 1 << bits
    fmask = [((1 << width[v]) - 1) << off[v] for v in range(n)]
    mb = [set() for _ in range(n)]
    for c in range(n):
        ps = onet.parents[c]
        for p in ps:
            mb[c].add(p)
            mb[p].add(c)
            for q in ps:
                if q != p:
                    mb[p].add(q)

    def fields(S):
        return [(S >> off[v]) & ((1 << width[v]) - 1) for v in range(n)]

    vprob = {}
    for v in range(n):
        for S in range(R):
            a = fields(S)
            if any(a[u] >= cards[u] for u in mb[v]):
                vprob[v, S] = [0.0] * cards[v]
            else:
                vprob[v, S] = _conditional(onet, cpts, v, a)
    out = {}
    for P in range(1, 1 << n):
        lm = 0
        for v in range(n):
            if (P >> v) & 1:
                lm |= fmask[v]
        pos = [i for i in range(bits) if (lm >> i) & 1]
        B = len(pos)
        K = 1 << B
        dep = [sum(((j >> i) & 1) << pos[i] for i in range(B)) for j in range(K)]
        keep = (R - 1) & ~lm
        rows = np.zeros((R, K), dtype=np.uint32)
        for S in range(R):
            prods = []
            for j in range(K):
                Sn = (S & keep) | dep[j]
                a = fields(Sn)
                cur = fields(S)
                p = 1.0
                for v in order:
                    if not (P >> v) & 1:
                        continue
                    if a[v] >= cards[v]:
                        p = 0.0
                        break
                    p = p * vprob[v, sum(cur[u] << off[u] for u in mb[v])][a[v]]
                    cur[v] = a[v]
                prods.append(p)
            cum = warp_scan(np.asarray(prods, dtype=np.float64))
            rows[S] = alias_row(cum, B)
        out[P] = (B, keep, np.asarray(dep, dtype=np.int64), rows)
    return out


def alias_row(cum, B):
    """Alias entries of one row (csrc joint_alias_row): integer masses
    w_j = C_j - C_{j-1}, C_j = min(ceil(cum_j * 2^32 / total), 2^32), C_{K-1} = 2^32;
    T = 2^(32-B); lights (w < T) and heavies (w > T) laid out in column order
    on a deficit and a surplus line; light: primary w, alias = the heavy whose
    surplus interval holds the light's start; heavy: overshoot = first light
    end >= its end E_h, minus E_h; primary T - overshoot and alias = next heavy
    when the overshoot is positive, else full; full columns alias themselves.
    Entry = primary << B | alias."""
    import math

    K = 1 << B
    total = float(cum[-1])
    sc = 4294967296.0 / total if total > 0.0 else 0.0
    def quant(c):  # fmin(ceil(c * sc), 2^32) as the device rounds it (NaN / inf -> 2^32)
        x = c * sc
        return 4294967296 if (math.isnan(x) or x >= 4294967296.0) else math.ceil(x)

    C = [quant(float(cum[j])) if j < K - 1 else 4294967296 for j in range(K)]
    w = [C[j] - (C[j - 1] if j else 0) for j in range(K)]
    T = 1 << (32 - B)
    d = [T - x if x < T else 0 for x in w]
    e = [x - T if x > T else 0 for x in w]
    Dinc = np.cumsum(d).tolist()
    Einc = np.cumsum(e).tolist()
    out = np.zeros(K, dtype=np.uint32)
    for j in range(K):
        if w[j] < T:
            alias = int(np.searchsorted(Einc, Dinc[j] - d[j], side="right"))
            out[j] = (w[j] << B) | alias
        elif w[j] > T:
            X = Dinc[int(np.searchsorted(Dinc, Einc[j], side="left"))]
            ov = X - Einc[j]
            out[j] = ((T - ov) << B) | int(np.searchsorted(Einc, Einc[j], side="right")) if ov else j
        else:
            out[j] = j
    return out


def alias_probs(entries, B):
    """Column probabilities an alias row encodes (x 2^32, exact integers)."""
    K = 1 << B
    T = 1 << (32 - B)
    p = [0] * K
    for i, e in enumerate(int(x) for x in entries):
        thr, al = e >> B, e & (K - 1)
        p[i] += thr
        p[al] += T - thr
    return p


def joint_sweep(tabs, cards, lanes_in, latent, key, case_base=0):
    """One joint sweep of generic lane states (n, m, cases) with latent mask
    (n, cases): lane (r, c) draws word u = r % 4 of the FAST block (case, 0,
    quad r // 4, purpose 2) and reads entry i = u >> (32 - B) of its alias
    row: column i when (u mod 2^(32-B)) < the entry's primary, else its alias."""
    width, off = lane_fields(cards)
    n, m, cases = lanes_in.shape
    S = np.zeros((m, cases), dtype=np.int64)
    for v in range(n):
        S |= lanes_in[v].astype(np.int64) << off[v]
    P = np.zeros(cases, dtype=np.int64)
    for v in range(n):
        P |= latent[v].astype(np.int64) << v
    gc = np.arange(cases, dtype=np.uint64) + np.uint64(case_base)
    out = S.copy()
    for r in range(m):
        u = fast_block(key, gc, 0, r >> 2, 2)[:, r & 3].astype(np.int64)
        for p in np.unique(P):
            if p == 0:
                continue
            B, keep, dep, rows = tabs[int(p)]
            sel = np.flatnonzero(P == p)
            i = u[sel] >> (32 - B)
            e = rows[S[r, sel], i].astype(np.int64)
            f = u[sel] & ((1 << (32 - B)) - 1)
            j = np.where(f < (e >> B), i, e & ((1 << B) - 1))
            out[r, sel] = (S[r, sel] & keep) | dep[j]
    res = np.zeros_like(lanes_in)
    for v in range(n):
        res[v] = (out >> off[v]) & ((1 << width[v]) - 1)
    return res
