"""The FAST stream's Philox4x32-10 restatement against Random123's published
known-answer vectors (CPU), and the device FAST stream against it (GPU)."""

import numpy as np
import pytest

from fast_stream import fast_init_states, philox4x32_10

# Random123 kat_vectors, philox4x32_10: counter, key -> output
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox4x32_10_known_answers(ctr, key, want):
    got = philox4x32_10(np.array(ctr, dtype=np.uint32), key)
    assert tuple(int(x) for x in got) == want


@pytest.mark.gpu
@pytest.mark.parametrize("case_base", [0, 3_000_000_000])
def test_device_fast_init_matches_restatement(case_base):
    """sg_init_states (FAST) = fast_init_states: the device Philox and counter
    layout are the documented ones, including the top of the 32-bit case range."""
    import torch

    import paper_1511_06416_b200 as sg
    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.device import netpack, stream_handle
    from paper_1511_06416_b200.sampler import DeviceBatch

    rng = np.random.default_rng(5)
    cards = [2, 3, 4, 2, 3]
    net = sg.build_network(cards, [(0, 1), (1, 2), (0, 3), (3, 4)])
    cases, m = 777, 7
    obs = np.where(rng.random((5, cases)) < 0.5, -1, rng.integers(0, 2, (5, cases))).astype(np.int8)
    pitch = (cases + 15) // 16 * 16
    dobs = torch.full((5, pitch), -1, dtype=torch.int8, device="cuda")
    dobs[:, :cases] = torch.from_numpy(obs).cuda()
    pack = netpack(net)
    db = DeviceBatch(5, m, cases, cases, torch.device("cuda"), case_base)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    key = 0x0123456789ABCDEF
    _lib.call("sg_init_states", pack.ref, db.ref, dobs.data_ptr(), pitch, _lib.SG_RNG_FAST, key, None, None,
              err.data_ptr(), stream_handle())
    torch.cuda.synchronize()
    got = db.states[:, :, :cases].cpu().numpy()
    np.testing.assert_array_equal(got, fast_init_states(key, obs, cards, m, case_base))
    assert int(err.item()) == 0
