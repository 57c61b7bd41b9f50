"""Host-side API behaviour that needs no GPU (reference tests/test_sampler.py
and tests/test_network.py pin the same): annealing schedules, configuration
validation, SAME replication of a minibatch, network validation and colouring."""

import numpy as np
import pytest

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.sampler import pad_block, replicate_minibatch


def test_anneal_schedule_pieces():
    assert sg.anneal_m(((1, 50), (5, 150)), 10) == 1
    assert sg.anneal_m(((1, 50), (5, 150)), 60) == 5
    assert sg.anneal_m(5, 123) == 5 and sg.anneal_m(((5, 10),), 3) == 5
    assert sg.anneal_m(((1, 5), (7, 5)), 1000) == 7
    with pytest.raises(ValueError):
        sg.anneal_m((), 0)
    with pytest.raises(ValueError):
        sg.anneal_m(3, -1)


@pytest.mark.parametrize("kw", [dict(accumulator_mode="exponential", exp_decay=0.0),
                                dict(accumulator_mode="decaying"), dict(same_m=0), dict(same_m=[(1, 0)]),
                                dict(rng="mersenne")])
def test_config_validation(kw):
    with pytest.raises(ValueError):
        sg.SamplerConfig(**kw)


def test_replication_shares_observed_cells():
    dense = np.array([[0, 1, -1, 0], [-1, 2, 1, -1]], dtype=np.int32)
    batch = replicate_minibatch(pad_block(0, dense, 4), 3)
    assert batch.num_lanes == 12
    for r in range(3):
        lane = batch.values[:, r * 4:(r + 1) * 4]
        np.testing.assert_array_equal(lane[dense >= 0], dense[dense >= 0])
    for v in range(2):  # latent lanes listed in the reference's lane order r*B + c
        want = [r * 4 + c for r in range(3) for c in range(4) if dense[v, c] < 0]
        np.testing.assert_array_equal(batch.missing_lanes[v], want)
    one = replicate_minibatch(pad_block(0, dense[:1], 4), 1)
    np.testing.assert_array_equal(one.values, dense[:1])


def test_padding_has_zero_weight():
    mb = pad_block(2, np.array([[0, 1, 1]], dtype=np.int32), 8)
    assert mb.size == 8 and mb.num_real == 3
    np.testing.assert_array_equal(mb.weights, [1, 1, 1, 0, 0, 0, 0, 0])
    assert (np.asarray(mb.values)[:, 3:] == -1).all()


@pytest.mark.parametrize("cards,edges,err", [
    ([2, 2], [(0, 1), (1, 0)], "CycleDetected"),
    ([2, 2], [(0, 2)], "InvalidIndex"),
    ([2, 2], [(0, 1), (0, 1)], "DuplicateEdge"),
    ([1, 2], [(0, 1)], "CardinalityTooSmall"),
])
def test_network_validation_errors(cards, edges, err):
    with pytest.raises(getattr(sg, err)):
        sg.build_network(cards, edges)


def test_colouring_is_proper_and_covers_every_variable():
    from paper_1511_06416_b200 import netgen

    net = netgen.random_dag_network(200, max_parents=4, seed=9)
    g = sg.moralize(net)
    col = sg.color_graph(g)
    colour = {v: k for k, grp in enumerate(col.groups) for v in grp}
    assert sorted(colour) == list(range(net.num_vars))
    for a, b in g.edges:
        assert colour[a] != colour[b]


@pytest.mark.parametrize("encoding", ["int8", "nibble"])
def test_sgb_writer_layout(tmp_path, encoding):
    """.sgb blocks hold the dense matrix column-block by column-block
    (4-bit: case 2j low nibble, 15 = missing)."""
    from paper_1511_06416_b200 import io

    rng = np.random.default_rng(3)
    dense = rng.integers(-1, 4, size=(3, 70)).astype(np.int32)
    path = tmp_path / "d.sgb"
    io.write_binary(path, dense, 40, encoding)
    h = io.read_binary_header(path)
    assert (h["num_vars"], h["num_cases"], h["block_cases"], h["pitch"]) == (3, 70, 40, 64)
    raw = np.fromfile(path, dtype=np.uint8, offset=64)
    rb = 64 if encoding == "int8" else 32
    blocks = raw.reshape(2, 3, rb)
    for b in range(2):
        want = np.full((3, 64), -1, dtype=np.int64)
        seg = dense[:, b * 40:(b + 1) * 40]
        want[:, :seg.shape[1]] = seg
        if encoding == "int8":
            got = blocks[b].view(np.int8).astype(np.int64)
        else:
            got = np.empty((3, 64), dtype=np.int64)
            got[:, 0::2] = blocks[b] & 15
            got[:, 1::2] = blocks[b] >> 4
            got[got == 15] = -1
        np.testing.assert_array_equal(got, want)
    with pytest.raises(ValueError):
        io.write_binary(tmp_path / "x.sgb", np.full((1, 4), 15), 4, "nibble")


def test_pack_nibbles_matches_sgb_blocks(tmp_path):
    """io.pack_nibbles (numpy and torch) is the 4-bit .sgb block layout."""
    import numpy as np
    import torch

    from paper_1511_06416_b200 import io

    rng = np.random.default_rng(3)
    dense = rng.integers(-1, 5, size=(4, 45)).astype(np.int32)
    io.write_binary(tmp_path / "a.sgb", dense, block_cases=45, encoding="nibble")
    h = io.read_binary_header(tmp_path / "a.sgb")
    raw = np.fromfile(tmp_path / "a.sgb", dtype=np.uint8)[64:].reshape(4, h["pitch"] // 2)
    np.testing.assert_array_equal(io.pack_nibbles(dense, h["pitch"]), raw)
    np.testing.assert_array_equal(io.pack_nibbles(torch.from_numpy(dense), h["pitch"]).numpy(), raw)


def test_pack_crumbs_matches_sgb_blocks(tmp_path):
    """io.pack_crumbs (2-bit) is the crumb .sgb block layout; the header round-trips."""
    import numpy as np

    from paper_1511_06416_b200 import io

    rng = np.random.default_rng(4)
    dense = rng.integers(-1, 3, size=(3, 70)).astype(np.int32)
    io.write_binary(tmp_path / "c.sgb", dense, block_cases=70, encoding="crumb")
    h = io.read_binary_header(tmp_path / "c.sgb")
    assert h["encoding"] == "crumb" and h["pitch"] == 128
    raw = np.fromfile(tmp_path / "c.sgb", dtype=np.uint8)[64:].reshape(3, h["pitch"] // 4)
    np.testing.assert_array_equal(io.pack_crumbs(dense, h["pitch"]), raw)
    x = raw[:, :18].astype(np.int64)  # decode by hand
    dec = np.stack([(x >> (2 * k)) & 3 for k in range(4)], axis=-1).reshape(3, -1)[:, :70]
    np.testing.assert_array_equal(np.where(dec == 3, -1, dec), dense)


def _bft_weights(start, desc, src, cpt, x, v):
    """Host restatement of draw_bft's weight product (sg_big.cu) from the plan."""
    def row_of(r):
        base, sk = int(src[2 * r]), int(src[2 * r + 1])
        step, k = sk & ((1 << 26) - 1), sk >> 26
        return np.array([cpt[base + t * step] if t < k else 0.0 for t in range(4)])

    p = int(start[v]) // 4
    rec = desc.reshape(-1, 4)
    card, npar, nchl, row = rec[p]
    p += 1
    for j in range(0, npar, 2):
        u0, s0, u1, s1 = rec[p]
        row += x[u0] * s0 + x[u1] * s1
        p += 1
    w = row_of(row)
    for _ in range(nchl):
        c, base, nrec, _z = rec[p]
        p += 1
        i = base + x[c]
        for _q in range(nrec):
            u0, s0, u1, s1 = rec[p]
            i += x[u0] * s0 + x[u1] * s1
            p += 1
        w = w * row_of(i)
    return w


def test_blanket_factor_plan_reproduces_the_weight_product():
    """Every row of the big-tile sweep's blanket factor tables is the CPT
    entry the reference's weight product (sampler.py:226-240) multiplies."""
    from paper_1511_06416_b200 import netgen, netpack

    net = netgen.random_dag_network(60, max_parents=4, min_card=2, max_card=4, seed=9)
    cpts = netgen.dirichlet_cpts(net, 1.0, seed=10)
    lay = netpack.layout(net)
    start, desc, src, rows = netpack.blanket_factor_plan(net, lay)
    assert rows == len(src) // 2
    cpt = np.concatenate([t.ravel() for t in cpts.tables])
    rng = np.random.default_rng(0)
    for _ in range(20):
        x = [int(rng.integers(k)) for k in net.cardinalities]
        for v in range(net.num_vars):
            ref = np.zeros(4)
            for t in range(net.cardinalities[v]):
                xs = list(x)
                xs[v] = t
                w = cpts.tables[v][sum(xs[p] * s for p, s in zip(net.parents[v], net.parent_strides(v))), t]
                for c in net.children[v]:
                    ci = sum(xs[p] * s for p, s in zip(net.parents[c], net.parent_strides(c)))
                    w = w * cpts.tables[c][ci, xs[c]]
                ref[t] = w
            np.testing.assert_array_equal(_bft_weights(start, desc, src, cpt, x, v), ref)
