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
