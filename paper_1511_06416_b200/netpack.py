"""Flatten a Network + colouring into the device arrays of ``sg_net``.

Host precompute, once per run (reference: ``_NetCache`` sampler.py:190-202,
``parent_strides`` network.py:42-48, ``color_graph(moralize(net))``
sampler.py:409).  Besides the reference's parent strides and child links it
derives each variable's Markov blanket and the blanket -> table index map
used by the conditional tables (sg_tables.cu).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import NET_POINTERS, NET_POINTERS_TAIL, SgNet
from .network import Coloring, Network, color_graph, moralize

# A variable's full conditional is tabulated when its blanket has at most this
# many configurations and the tables stay within the byte budget below; the
# others are evaluated per lane from the CPTs ("direct" variables).
# Conditional tables pay off only while the sweep can stage them in shared
# memory (n <= TABLE_MAX_VARS, parity table <= TABLE_BUDGET_BYTES): tables read
# from L2 lose to the factored weight product, and mixing the two draw kinds in
# one large network costs instruction-cache misses (measured on B200, C4
# shape: 39 ms factored-only vs 51 ms with 32 KB of tables vs 82 ms with 52 MB).
TABLE_MAX_ENTRIES = 1 << 16
TABLE_BUDGET_BYTES = 48 << 10
TABLE_MAX_VARS = 512
MAX_CARD = 64
MAX_MB = 64
JOINT_MAX = 128        # SG_JOINT_MAX
DESC_MB = 8            # SG_DESC_MB
DESC_WORDS = 4 + 2 * DESC_MB


@dataclass
class NetLayout:
    """Host-side (numpy) description; the device copy is built by :class:`NetPack`."""

    n: int
    cards: np.ndarray
    rows: np.ndarray
    cpt_off: np.ndarray      # [n+1] cell prefix
    row_off: np.ndarray      # [n+1]
    groups: tuple[tuple[int, ...], ...]
    topo: np.ndarray
    int32: dict[str, np.ndarray]
    int64: dict[str, np.ndarray]
    scalars: dict[str, int]

    @property
    def cells(self) -> int:
        return int(self.cpt_off[-1])


def layout(net: Network, coloring: Coloring | None = None,
           table_max_entries: int | None = None,
           table_budget_bytes: int | None = None) -> NetLayout:
    n = net.num_vars
    table_max_entries = TABLE_MAX_ENTRIES if table_max_entries is None else table_max_entries
    table_budget_bytes = TABLE_BUDGET_BYTES if table_budget_bytes is None else table_budget_bytes
    if coloring is None:
        coloring = color_graph(moralize(net))
    cards = np.asarray(net.cardinalities, dtype=np.int64)
    if n and cards.max() > MAX_CARD:
        raise ValueError(f"cardinality {int(cards.max())} exceeds the device limit {MAX_CARD}")
    rows = np.array([net.num_parent_configs(v) for v in range(n)], dtype=np.int64)
    cpt_off = np.zeros(n + 1, dtype=np.int64)
    cpt_off[1:] = np.cumsum(rows * cards)
    row_off = np.zeros(n + 1, dtype=np.int64)
    row_off[1:] = np.cumsum(rows)


    par_start, par_var, par_stride, par_slot = [0], [], [], []
    mb_start, mb_var, mb_stride = [0], [], []
    chl_start, chl_var, chl_vstride, chl_slot = [0], [], [], []
    chl_pstart, chl_pslot, chl_pstride = [0], [], []
    mb_sizes, mb_confs = [], []
    blankets = []
    for v in range(n):
        blanket = set(net.parents[v]) | set(net.children[v])
        for c in net.children[v]:
            blanket |= set(net.parents[c])
        blanket.discard(v)
        mb = sorted(blanket)
        if len(mb) > MAX_MB:
            raise ValueError(f"Markov blanket of variable {v} has {len(mb)} members (limit {MAX_MB})")
        blankets.append(mb)
        slot = {u: k for k, u in enumerate(mb)}
        strides = []
        acc = 1
        for u in reversed(mb):
            strides.append(acc)
            acc = acc * int(cards[u])
        strides.reverse()
        confs = acc
        mb_confs.append(confs)
        mb_sizes.append(len(mb))
        mb_var.extend(mb)
        # strides of huge blankets are meaningless (direct variables); clamp to int32
        mb_stride.extend(min(s, 2**31 - 1) for s in strides)
        mb_start.append(len(mb_var))
        ps = net.parent_strides(v)
        for j, p in enumerate(net.parents[v]):
            par_var.append(p)
            par_stride.append(int(ps[j]))
            par_slot.append(slot[p])
        par_start.append(len(par_var))
        for c in net.children[v]:
            cps = net.parent_strides(c)
            j = net.parents[c].index(v)
            chl_var.append(c)
            chl_vstride.append(int(cps[j]))
            chl_slot.append(slot[c])
            for q, p in enumerate(net.parents[c]):
                if p != v:
                    chl_pslot.append(slot[p])
                    chl_pstride.append(int(cps[q]))
            chl_pstart.append(len(chl_pslot))
        chl_start.append(len(chl_var))

    # choose tabulated variables: smallest tables first under the byte budget
    tab_entries = np.zeros(n, dtype=np.int64)
    budget = table_budget_bytes
    for v in sorted(range(n), key=lambda v: mb_confs[v]) if n <= TABLE_MAX_VARS else ():
        e = mb_confs[v]
        nbytes = e * int(cards[v]) * 8
        if e <= table_max_entries and nbytes <= budget:
            tab_entries[v] = e
            budget -= nbytes
    tab_start = np.zeros(n + 1, dtype=np.int64)
    tab_start[1:] = np.cumsum(tab_entries)

    # Inside a colour group the order is result-neutral (the members are
    # conditionally independent and draw from per-variable streams).  The sweep
    # compacts latent cells variable-major and a warp takes 32 consecutive
    # items, so members with the same draw kind (table with k blanket members,
    # or the factored product) sit together, costliest first.
    def kind(v):
        k = len(blankets[v]) if tab_entries[v] > 0 and len(blankets[v]) <= DESC_MB else DESC_MB + 1
        return (k, -(len(net.children[v]) + len(net.parents[v])), v)

    order = [v for grp in coloring.groups for v in sorted(grp, key=kind)]
    group_start = np.zeros(len(coloring.groups) + 1, dtype=np.int64)
    group_start[1:] = np.cumsum([len(g) for g in coloring.groups])
    ptab_len = tab_entries * cards
    ftab_len = tab_entries * (cards - 1)
    ptab_off = np.zeros(n, dtype=np.int64)
    ftab_off = np.zeros(n, dtype=np.int64)
    if n:
        ptab_off[1:] = np.cumsum(ptab_len)[:-1]
        ftab_off[1:] = np.cumsum(ftab_len)[:-1]
    row_var = np.repeat(np.arange(n, dtype=np.int64), rows)

    # compact draw descriptors (sg_sweep): card, nmb | -1, ftab off, ptab off, mb vars, mb strides
    desc = np.zeros((n, DESC_WORDS), dtype=np.int64)
    for v in range(n):
        mb = blankets[v]
        desc[v, 0] = cards[v]
        if tab_entries[v] > 0 and len(mb) <= DESC_MB:
            desc[v, 1] = len(mb)
            desc[v, 2] = ftab_off[v]
            desc[v, 3] = ptab_off[v]
            desc[v, 4:4 + len(mb)] = mb
            desc[v, 4 + DESC_MB:4 + DESC_MB + len(mb)] = mb_stride[mb_start[v]:mb_start[v + 1]]
        else:
            desc[v, 1] = -1
    # factored draw descriptors (draw_factored, sg_sweep.cu): the reference's
    # weight product (sampler.py:226-240) with every index pre-multiplied:
    #   card, npar, nchl, cpt_off[v],
    #   npar x (parent, stride * card),
    #   nchl x (child, cpt_off[c], card[c], vstride * card[c], nq, 0, nq x (other parent, stride * card[c]))
    fac_start, fac = [0], []
    for v in range(n):
        card = int(cards[v])
        ps = net.parent_strides(v)
        fac += [card, len(net.parents[v]), len(net.children[v]), int(cpt_off[v])]
        for j, p in enumerate(net.parents[v]):
            fac += [p, int(ps[j]) * card]
        for c in net.children[v]:
            cps = net.parent_strides(c)
            cc = int(cards[c])
            j = net.parents[c].index(v)
            others = [(p, int(cps[q]) * cc) for q, p in enumerate(net.parents[c]) if p != v]
            fac += [c, int(cpt_off[c]), cc, int(cps[j]) * cc, len(others), 0]  # 6 words: pairs stay 8-byte aligned
            for p, st in others:
                fac += [p, st]
        fac_start.append(len(fac))

    # chunked tally: runs of consecutive variables whose cells fit one
    # shared-memory histogram (SG_TALLY_CHUNK_CELLS)
    from ._lib import TALLY_CHUNK_CELLS

    tally_chunk = [0]
    acc = 0
    for v in range(n):
        c = int(rows[v] * cards[v])
        if acc and acc + c > TALLY_CHUNK_CELLS:
            tally_chunk.append(v)
            acc = 0
        acc += c
    if n:
        tally_chunk.append(n)

    # joint-state tally tables (small networks)
    joint = int(np.prod(cards)) if n else 0
    if 0 < joint <= JOINT_MAX:
        radix = np.ones(n, dtype=np.int64)
        for v in range(n - 2, -1, -1):
            radix[v] = radix[v + 1] * cards[v + 1]
        states = (np.arange(joint)[:, None] // radix[None, :]) % cards[None, :]
        jcell = np.zeros((joint, n), dtype=np.int64)
        for v in range(n):
            cfg = np.zeros(joint, dtype=np.int64)
            for p, s in zip(net.parents[v], net.parent_strides(v)):
                cfg += states[:, p] * int(s)
            jcell[:, v] = cpt_off[v] + cfg * cards[v] + states[:, v]
    else:
        joint = 0
        radix = np.zeros(1, dtype=np.int64)
        jcell = np.zeros((1, 1), dtype=np.int64)

    def i32(x):
        a = np.asarray(x, dtype=np.int64)
        if a.size and (a.max() > 2**31 - 1 or a.min() < -2**31):
            raise ValueError("index overflow in network pack")
        return a.astype(np.int32)

    int32 = {
        "card": i32(cards), "group_start": i32(group_start), "order": i32(order),
        "par_start": i32(par_start), "par_var": i32(par_var), "par_stride": i32(par_stride),
        "par_slot": i32(par_slot), "mb_start": i32(mb_start), "mb_var": i32(mb_var),
        "mb_stride": i32(mb_stride), "chl_start": i32(chl_start), "chl_var": i32(chl_var),
        "chl_vstride": i32(chl_vstride), "chl_slot": i32(chl_slot), "chl_pstart": i32(chl_pstart),
        "chl_pslot": i32(chl_pslot), "chl_pstride": i32(chl_pstride), "row_var": i32(row_var),
        "joint_radix": i32(radix), "joint_cell": i32(jcell.ravel()), "var_desc": i32(desc.ravel()),
        "fac_start": i32(fac_start), "fac_desc": i32(fac), "tally_chunk": i32(tally_chunk),
    }
    int64 = {
        "cpt_off": cpt_off[:n].copy(), "row_off": row_off, "tab_entries": tab_entries,
        "tab_start": tab_start, "ptab_off": ptab_off, "ftab_off": ftab_off,
    }
    scalars = {
        "n": n,
        "num_groups": len(coloring.groups),
        "max_card": int(cards.max()) if n else 0,
        "max_mb": max(mb_sizes) if n else 0,
        "max_group": max((len(g) for g in coloring.groups), default=0),
        "direct_vars": int((tab_entries == 0).sum()),
        "cells": int(cpt_off[-1]),
        "rows": int(row_off[-1]),
        "ptab_size": int(ptab_len.sum()),
        "ftab_size": int(ftab_len.sum()),
        "table_entries": int(tab_entries.sum()),
        "joint_size": joint,
        "tally_chunks": len(tally_chunk) - 1,
    }
    return NetLayout(n=n, cards=cards, rows=rows, cpt_off=cpt_off, row_off=row_off,
                     groups=coloring.groups, topo=np.asarray(net.topo_order, dtype=np.int32),
                     int32=int32, int64=int64, scalars=scalars)


BFT_MIN_VARS = 33  # the big-tile sweep's networks (sg_big.cu: n > 32)


def blanket_factor_plan(net: Network, lay: NetLayout):
    """Blanket factor tables of the big-tile sweep (sg_big.cu, cards <= 4).

    Every factor of v's weight product (sampler.py:226-240) -- v's own CPT row
    and, per child c, c's CPT entry as v runs over its states -- becomes one
    row of 4 doubles (states of v, zero padded), so a draw gathers one
    contiguous 32-byte row per factor instead of card strided cells.  Rows are
    exact copies of CPT cells (``k_build_bft`` refreshes them from the CPTs at
    each large-network sweep), so the product and every draw are unchanged.

    Returns ``(start, desc, src, rows)`` or None:
      desc at start[v] (int4 records): [card, npar, nchl, own row base];
        ceil(npar/2) x [u, stride, u, stride] (own row += x_u * stride);
        per child: [c, row base, nrec, 0] + nrec x [u, stride, u, stride]
        (row = base + x_c + sum x_u * stride; unused halves have stride 0);
      src[row] = [first CPT cell, cell step | card_v << 26].
    """
    n = net.num_vars
    cards = lay.cards
    if n < BFT_MIN_VARS or int(cards.max()) > 4:
        return None
    cpt_off = lay.cpt_off
    start, desc, src = [0], [], []
    rows = 0

    def records(pairs):
        out = []
        for i in range(0, len(pairs), 2):
            (u0, s0), (u1, s1) = pairs[i], pairs[i + 1] if i + 1 < len(pairs) else (pairs[i][0], 0)
            out += [u0, s0, u1, s1]
        return out

    for v in range(n):
        kv = int(cards[v])
        ps = net.parent_strides(v)
        nrow = int(lay.rows[v])
        desc += [kv, len(net.parents[v]), len(net.children[v]), rows]
        desc += records([(p, int(ps[j])) for j, p in enumerate(net.parents[v])])
        r = np.arange(nrow, dtype=np.int64)
        src.append(np.stack([cpt_off[v] + r * kv, np.full(nrow, 1 | (kv << 26), np.int64)], 1))
        rows += nrow
        for c in net.children[v]:
            cc = int(cards[c])
            cps = net.parent_strides(c)
            j = net.parents[c].index(v)
            others = [(q, p) for q, p in enumerate(net.parents[c]) if p != v]
            # reduced mixed radix over the other parents (first most significant), x_c innermost
            red = [1] * len(others)
            for i in range(len(others) - 2, -1, -1):
                red[i] = red[i + 1] * int(cards[others[i + 1][1]])
            recs = records([(p, red[i] * cc) for i, (q, p) in enumerate(others)])
            desc += [c, rows, len(recs) // 4, 0] + recs
            nconf = int(np.prod([int(cards[p]) for _, p in others])) if others else 1
            # row o * cc + x_c: cells cpt_off[c] + (sum_q x_q cps[q] + t cps[j]) * cc + x_c
            o = np.arange(nconf, dtype=np.int64)
            full = np.zeros(nconf, dtype=np.int64)
            for i, (q, p) in enumerate(others):
                full += ((o // red[i]) % int(cards[p])) * int(cps[q])
            first = cpt_off[c] + (full[:, None] * cc + np.arange(cc)[None, :]).ravel()
            step = int(cps[j]) * cc
            if step >= 1 << 26:
                return None
            src.append(np.stack([first, np.full(first.size, step | (kv << 26), np.int64)], 1))
            rows += first.size
        start.append(len(desc))
    if rows >= 2**31 or cpt_off[-1] >= 2**31:
        return None
    return (np.asarray(start, np.int32), np.asarray(desc, np.int32),
            np.concatenate(src).astype(np.int32).ravel(), rows)


def small_plan(net: Network, lay: NetLayout):
    """Packed-lane plan (``sg_small``) when the lane state fits in one byte.

    Returns ``(SgSmall, jcell)`` or None.  Field widths are ceil(log2(card));
    jcell[S, v] is the CPT cell variable v contributes to for lane word S.
    """
    from ._lib import SMALL_MAXBITS, SMALL_MAXV, SgSmall

    n = net.num_vars
    if n == 0 or n > SMALL_MAXV:
        return None
    cards = [int(k) for k in net.cardinalities]
    if max(cards) > 4 or min(cards) < 2:  # one aligned LDS / LDS.64 / LDS.128 of 1..3 thresholds per draw
        return None
    width = [max(1, (k - 1).bit_length()) for k in cards]
    bits = sum(width)
    if bits > SMALL_MAXBITS:
        return None
    off = [0] * n
    for v in range(1, n):
        off[v] = off[v - 1] + width[v - 1]
    mb_start = lay.int32["mb_start"]
    mb_var = lay.int32["mb_var"]
    sp = SgSmall()
    sp.n, sp.bits = n, bits
    order = [v for grp in lay.groups for v in grp]
    # entries padded to 1, 2 or 4 words (card-1 thresholds) so a lookup is one
    # aligned LDS / LDS.64 / LDS.128; tables aligned to their entry size
    toff, tstride, words = [], [], 0
    for v in range(n):
        k1 = cards[v] - 1
        stride = 1 if k1 == 1 else 2 if k1 == 2 else 4 if k1 <= 4 else k1
        words = (words + stride - 1) // stride * stride if stride in (2, 4) else words
        toff.append(words)
        tstride.append(stride)
        words += (1 << bits) * stride
    sp.tab_words = words
    for v in range(n):
        sp.order[v] = order[v]
        sp.off[v] = off[v]
        sp.width[v] = width[v]
        sp.card[v] = cards[v]
        sp.toff[v] = toff[v]
        sp.tstride[v] = tstride[v]
        mask = 0
        for u in mb_var[mb_start[v]:mb_start[v + 1]]:
            mask |= ((1 << width[u]) - 1) << off[u]
        sp.mbmask[v] = mask
    S = np.arange(1 << bits)
    fields = np.stack([(S >> off[v]) & ((1 << width[v]) - 1) for v in range(n)], axis=1)
    valid = (fields < np.asarray(cards)[None, :]).all(axis=1)
    jcell = np.zeros((1 << bits, n), dtype=np.int64)
    for v in range(n):
        cfg = np.zeros(1 << bits, dtype=np.int64)
        for p, st in zip(net.parents[v], net.parent_strides(v)):
            cfg += fields[:, p] * int(st)
        jcell[:, v] = np.where(valid, lay.cpt_off[v] + cfg * cards[v] + fields[:, v], 0)
    return sp, jcell.astype(np.int32)


JOINT_MAXB = 6           # lane words of <= 6 bits (csrc/sg_small.cu SG_JOINT_MAXB)
JOINT_THREADS = 1024     # SG_JOINT_THREADS
JOINT_SMEM_LIMIT = 227 * 1024


def joint_plan(sp, cells: int):
    """Static header of the joint-sweep blob (include/samegibbs_b200.h sg_joint).

    Patterns P (bit v = variable v latent, as sg_small_prepare buckets them):
    B_P latent bits, keep_P = the observed bits of the lane word, dep_P[j] =
    the lane bits of compact column j (bit i of j -> the i-th set bit of the
    latent mask), 2^bits rows of 2^B_P alias entries, 2^B_P + 1 words apart.  Returns ``(SgJoint,
    header uint32 array)`` or None when the network does not qualify or the
    CTA's shared memory (blob + per-variable table + per-warp tally bins) does not
    fit.
    """
    from ._lib import SgJoint

    if sp is None or not 2 <= sp.bits <= JOINT_MAXB:
        return None
    n, bits = sp.n, sp.bits
    NP = 1 << n
    fmask = [((1 << sp.width[v]) - 1) << sp.off[v] for v in range(n)]
    full = (1 << bits) - 1
    lmask = [0] * NP
    for P in range(NP):
        for v in range(n):
            if (P >> v) & 1:
                lmask[P] |= fmask[v]
    B = [bin(lm).count("1") for lm in lmask]
    dep, dep_off = [], [0] * NP
    for P in range(NP):
        if not B[P]:
            continue
        dep_off[P] = 2 * NP + len(dep)
        pos = [i for i in range(bits) if (lmask[P] >> i) & 1]
        for j in range(1 << B[P]):
            dep.append(sum(((j >> i) & 1) << pos[i] for i in range(B[P])))
    header_words = (2 * NP + len(dep) + 3) // 4 * 4
    row_off, words = [0] * NP, header_words
    for P in range(NP):
        if B[P]:  # rows 2^B + 1 words apart: odd stride, no bank conflicts between lanes
            row_off[P] = words
            words += (1 << bits) * ((1 << B[P]) + 1)
    words = (words + 3) // 4 * 4
    if max(dep_off) * 4 >= 1 << 16:
        return None
    head = np.zeros(header_words, dtype=np.uint32)
    for P in range(NP):
        head[P] = row_off[P] * 4
        head[NP + P] = B[P] | ((full & ~lmask[P]) << 8) | ((dep_off[P] * 4) << 16)
    head[2 * NP:2 * NP + len(dep)] = dep
    jp = SgJoint()
    jp.words, jp.header_words, jp.patterns, jp.max_b = words, header_words, NP, max(B)
    smem = (words * 4 + ((sp.tab_words * 4 + 15) & ~15) + (JOINT_THREADS // 32) * 65 * 4
            + ((cells * 4 + 15) & ~15) + 16)
    if smem > JOINT_SMEM_LIMIT:
        return None
    return jp, head


class NetPack:
    """Device-resident ``sg_net``: two flat tensors plus the C struct of pointers."""

    def __init__(self, net: Network, device: torch.device, coloring: Coloring | None = None, **kw):
        self.net = net
        self.layout = lay = layout(net, coloring, **kw)
        self.device = device
        self._views: dict[str, torch.Tensor] = {}
        offs32, offs64 = {}, {}
        parts32, parts64 = [], []
        pos = 0
        for k, a in lay.int32.items():
            # every array starts on a 16-byte boundary (vector loads of descriptors)
            a = a if len(a) else np.zeros(1, np.int32)
            a = np.concatenate([a, np.zeros((-len(a)) % 4, np.int32)])
            offs32[k] = pos
            pos += len(a)
            parts32.append(a)
        pos64 = 0
        for k, a in lay.int64.items():
            offs64[k] = pos64
            pos64 += max(len(a), 1)
            parts64.append(a if len(a) else np.zeros(1, np.int64))
        self.buf32 = torch.from_numpy(np.concatenate(parts32)).to(device)
        self.buf64 = torch.from_numpy(np.concatenate(parts64)).to(device)
        self.topo = torch.from_numpy(lay.topo).to(device)
        s = SgNet()
        for k, v in lay.scalars.items():
            setattr(s, k, v)
        for k in NET_POINTERS + NET_POINTERS_TAIL + ("tally_chunk",):
            if k in offs32:
                setattr(s, k, self.buf32.data_ptr() + 4 * offs32[k])
            else:
                setattr(s, k, self.buf64.data_ptr() + 8 * offs64[k])
        s.blob32, s.blob32_words = self.buf32.data_ptr(), self.buf32.numel()
        s.blob64, s.blob64_words = self.buf64.data_ptr(), self.buf64.numel()
        self.bft = None
        bplan = blanket_factor_plan(net, lay)
        if bplan is not None:
            start, desc, src, rows = bplan
            self.bft_prog = torch.from_numpy(np.concatenate([desc, start])).to(device)
            self.bft_src = torch.from_numpy(src).to(device)
            self.bft = torch.zeros(rows * 4, dtype=torch.float64, device=device)
            s.bft_rows = rows
            s.bft_desc = self.bft_prog.data_ptr()
            s.bft_start = self.bft_prog.data_ptr() + 4 * len(desc)
            s.bft_src = self.bft_src.data_ptr()
            s.bft = self.bft.data_ptr()
        self.struct = s
        self.ref = ctypes.byref(self.struct)
        plan = small_plan(net, lay)
        self.small = None
        if plan is not None:
            sp, jcell = plan
            self.small = sp
            self.small_ref = ctypes.byref(sp)
            self.small_jcell = torch.from_numpy(jcell.ravel()).to(device)
        self.joint = None
        jplan = joint_plan(self.small, lay.cells)
        if jplan is not None:
            self.joint, self.joint_header = jplan
            self.joint_ref = ctypes.byref(self.joint)

    def private_ref(self):
        """A copy of the ``sg_net`` struct with its own blanket-factor scratch
        (``bft``): what an engine passes to ``sg_sweep`` so that sweeps of one
        cached pack on different streams never share the scratch they rebuild.
        Returns ``(ctypes reference, keep-alive tuple)``."""
        s = SgNet()
        ctypes.memmove(ctypes.addressof(s), ctypes.addressof(self.struct), ctypes.sizeof(SgNet))
        bft = None
        if self.bft is not None:
            bft = torch.zeros_like(self.bft)
            s.bft = bft.data_ptr()
        return ctypes.byref(s), (s, bft)

    @property
    def n(self) -> int:
        return self.layout.n

    @property
    def cells(self) -> int:
        return self.layout.cells

    def flatten(self, tables) -> np.ndarray:
        """Concatenate per-variable tables (CptSet/CountSet order) into one fp64 vector."""
        if len(tables) != self.n:
            raise ValueError("table count does not match the network")
        out = np.empty(self.cells, dtype=np.float64)
        for v, t in enumerate(tables):
            a, b = self.layout.cpt_off[v], self.layout.cpt_off[v + 1]
            t = np.asarray(t, dtype=np.float64)
            if t.size != b - a:
                raise ValueError(f"table {v} has {t.size} cells, expected {b - a}")
            out[a:b] = t.ravel()
        return out

    def split(self, flat: np.ndarray) -> list[np.ndarray]:
        lay = self.layout
        return [flat[lay.cpt_off[v]:lay.cpt_off[v + 1]].reshape(int(lay.rows[v]), int(lay.cards[v])).copy()
                for v in range(self.n)]


class TablePack:
    """``sg_net`` carrying only the row layout of a table set (shapes).

    The row-wise kernels (sg_mean_cpts, sg_sample_cpts) read nothing but
    card / cpt_off / row_off / row_var, so a bare CountSet can be processed
    without its network (the reference's mean_cpts/sample_cpts take none).
    """

    _cache: dict = {}

    def __init__(self, shapes, device: torch.device):
        n = len(shapes)
        rows = np.array([r for r, _ in shapes], dtype=np.int64)
        cards = np.array([k for _, k in shapes], dtype=np.int64)
        if n and cards.max() > MAX_CARD:
            raise ValueError(f"cardinality {int(cards.max())} exceeds the device limit {MAX_CARD}")
        cpt_off = np.zeros(n + 1, dtype=np.int64)
        cpt_off[1:] = np.cumsum(rows * cards)
        row_off = np.zeros(n + 1, dtype=np.int64)
        row_off[1:] = np.cumsum(rows)
        self.cpt_off, self.rows, self.cards = cpt_off, rows, cards
        self.card_t = torch.from_numpy(cards.astype(np.int32)).to(device)
        self.rowvar_t = torch.from_numpy(np.repeat(np.arange(n, dtype=np.int32), rows)).to(device)
        self.off_t = torch.from_numpy(np.concatenate([cpt_off[:n], row_off])).to(device)
        s = SgNet()
        s.n = n
        s.max_card = int(cards.max()) if n else 0
        s.cells = int(cpt_off[-1])
        s.rows = int(row_off[-1])
        s.card = self.card_t.data_ptr()
        s.row_var = self.rowvar_t.data_ptr()
        s.cpt_off = self.off_t.data_ptr()
        s.row_off = self.off_t.data_ptr() + 8 * n
        self.struct = s
        self.ref = ctypes.byref(s)

    @classmethod
    def get(cls, shapes, device: torch.device) -> "TablePack":
        key = (shapes, device.index)
        pack = cls._cache.get(key)
        if pack is None:
            pack = cls._cache[key] = cls(shapes, device)
        return pack

    @property
    def n(self) -> int:
        return len(self.rows)

    @property
    def cells(self) -> int:
        return int(self.cpt_off[-1])

    def flatten(self, tables) -> np.ndarray:
        return np.concatenate([np.asarray(t, dtype=np.float64).ravel() for t in tables]) if tables else \
            np.zeros(0)

    def split(self, flat: np.ndarray) -> list[np.ndarray]:
        return [flat[self.cpt_off[v]:self.cpt_off[v + 1]].reshape(int(self.rows[v]), int(self.cards[v])).copy()
                for v in range(self.n)]
