"""predict_missing (reference metrics.py:89-139) on the device.

* bit-exact: with frozen CPTs and the numpy stream, the state frequencies
  equal the reference's own output (tests/golden/predict_c10.npz, made by
  tests/golden/make_acceptance.py on the c10 network);
* acceptance c10 (test_acceptance.py:287-306): held-out AUC after 100
  training passes beats the AUC after 10 passes, and each AUC is within
  AUC_TOL of the reference's own c10 AUC.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")

from golden_io import load  # noqa: E402

AUC_TOL = 0.03


def _problem():
    d = load("predict_c10")
    cards = [int(c) for c in d["cards"]]
    net = sg.build_network(cards, [tuple(int(x) for x in e) for e in d["edges"]])
    cpts = sg.CptSet([d[f"cpt_{i}"] for i in range(net.num_vars)])
    context = sg.DataMatrix.from_dense(d["context"])
    targets = [tuple(int(x) for x in t) for t in d["targets"]]
    return d, net, cpts, context, targets


def test_predict_missing_bit_exact_vs_reference():
    d, net, cpts, context, targets = _problem()
    freq = sg.predict_missing(net, cpts, context, targets, num_samples=int(d["num_samples"]), seed=int(d["seed"]),
                              burn_in=int(d["burn_in"]))
    assert freq.shape == d["freq"].shape
    np.testing.assert_array_equal(freq, d["freq"])


def test_predict_missing_edge_cases():
    d, net, cpts, context, targets = _problem()
    out = sg.predict_missing(net, cpts, context, [], num_samples=3, seed=1)
    assert out.shape[0] == 0
    with pytest.raises(ValueError):
        sg.predict_missing(net, cpts, context, targets[:3], num_samples=0, seed=1)
    with pytest.raises(sg.DimensionMismatch):
        sg.predict_missing(sg.build_network([2, 2], [(0, 1)]), sg.CptSet([np.full((1, 2), .5), np.full((2, 2), .5)]),
                           context, targets[:3], num_samples=1, seed=1)
    # frequencies are a distribution per target
    freq = sg.predict_missing(net, cpts, context, targets[:50], num_samples=7, seed=2, burn_in=1)
    np.testing.assert_allclose(freq.sum(axis=1), 1.0)
    assert np.all(freq * 7 == np.round(freq * 7))


def test_c10_roc_improves_with_training():
    d, net, _, train_set, targets = _problem()
    labels = d["labels"]
    aucs = {}
    for passes in (10, 100):
        cfg = sg.SamplerConfig(minibatch_size=2000, num_passes=passes, seed=14)
        cpts, _ = sg.run(net, train_set, cfg)
        probs = sg.predict_missing(net, cpts, train_set, targets, num_samples=300, seed=15, burn_in=30)
        aucs[passes] = sg.roc_auc(probs[:, 1], labels).auc
    print(f"c10 auc ours 10: {aucs[10]:.4f} 100: {aucs[100]:.4f}; reference {float(d['auc_10']):.4f} "
          f"{float(d['auc_100']):.4f}")
    assert aucs[100] > aucs[10]
    assert abs(aucs[10] - float(d["auc_10"])) <= AUC_TOL
    assert abs(aucs[100] - float(d["auc_100"])) <= AUC_TOL
