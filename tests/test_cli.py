"""The device backend of `samegibbs train` (reference cli.py:112-165): flags,
outputs, manifest replay, exit codes; the text I/O it reads.  CPU tests cover
the parser, the text formats and the error paths; the GPU test runs train on
the reference's coordinate file and on an .sgb file and checks the result
against the oracle (numpy stream + MAP: bit-exact)."""

import json

import numpy as np
import pytest

import oracle as O


def _koller_data(n=600, seed=3):
    onet, otruth = O.koller()
    dense = O.mask_dense(O.forward_sample(onet, otruth, n, seed), 0.5, seed + 1)
    return onet, otruth, dense


def test_text_data_round_trip(tmp_path):
    from paper_1511_06416_b200 import io
    from paper_1511_06416_b200.datagen import DataMatrix

    _, _, dense = _koller_data()
    dm = DataMatrix.from_dense(dense)
    io.write_data(tmp_path / "d.mm", dm)
    back = io.read_data(tmp_path / "d.mm")
    np.testing.assert_array_equal(back.to_dense(), dense)
    (tmp_path / "bad.mm").write_text("5 3 2\n1 1 1\n")
    with pytest.raises(io.ParseError):
        io.read_data(tmp_path / "bad.mm")


def test_text_format_matches_reference_writer(tmp_path):
    """Byte-compatible with the reference's write_data (io.py:105-116): header, 1-based triples."""
    from paper_1511_06416_b200 import io
    from paper_1511_06416_b200.datagen import DataMatrix

    dm = DataMatrix.from_dense(np.array([[0, -1, 2], [1, 1, -1]]))
    io.write_data(tmp_path / "d.mm", dm)
    assert (tmp_path / "d.mm").read_text() == "2 3 4\n1 1 1\n2 1 2\n2 2 2\n1 3 3\n"


def test_cli_validation_errors_exit_2(tmp_path):
    from paper_1511_06416_b200.cli import main

    assert main(["train", "--out", str(tmp_path / "o")]) == 2  # no --network / --data
    assert main(["train", "--network", "koller", "--data", str(tmp_path / "missing.mm"),
                 "--out", str(tmp_path / "o")]) == 2
    assert main(["train", "--network", "koller", "--data", "x", "--same-m", "3", "--same-schedule", "1x2",
                 "--out", str(tmp_path / "o")]) == 2
    assert main(["train", "--backend", "tpu", "--out", "o"]) == 2  # argparse rejects the choice


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["text", "sgb"])
def test_cli_train_matches_oracle(tmp_path, fmt):
    from paper_1511_06416_b200 import io
    from paper_1511_06416_b200.cli import main
    from paper_1511_06416_b200.datagen import DataMatrix

    onet, otruth, dense = _koller_data()
    data = tmp_path / ("d.mm" if fmt == "text" else "d.sgb")
    if fmt == "text":
        io.write_data(data, DataMatrix.from_dense(dense))
    else:
        io.write_binary(data, dense, 200, "nibble")
    out = tmp_path / "run"
    args = ["train", "--backend", "cuda", "--network", "koller", "--truth", "koller", "--data", str(data),
            "--out", str(out), "--minibatch-size", "200", "--passes", "3", "--same-m", "2", "--map-estimate",
            "--seed", "9"]
    assert main(args) == 0
    _, cpts = io.load_network_file(out / "cpts.json")
    ref = O.run(onet, dense, same_m=2, minibatch_size=200, num_passes=3, map_estimate=True, seed=9, truth=otruth)
    for a, b in zip(cpts.tables, ref.cpts):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-15)  # through the JSON text round trip
    trace = io.read_trace(out / "trace.csv")
    assert [r.kl_avg for r in trace.records] == ref.kl
    man = json.loads((out / "manifest.json").read_text())
    assert man["backend"] == "cuda" and man["passes"] == 3
    # replay from the manifest reproduces the run
    out2 = tmp_path / "replay"
    assert main(["train", "--from-manifest", str(out / "manifest.json"), "--out", str(out2)]) == 0
    assert (out2 / "cpts.json").read_text() == (out / "cpts.json").read_text()
