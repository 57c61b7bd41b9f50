"""Dev tool: time the generic sweep with / without the tally on a BASELINE shape."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import _lib
from paper_1511_06416_b200.engine import Engine
from paper_1511_06416_b200.device import stream_handle

import paper_1511_06416_b200.netpack as NP
import paper_1511_06416_b200.device as DV
args = [a for a in sys.argv[1:] if not a.startswith("--")]
for a in sys.argv[1:]:
    if a.startswith("--tmax="):
        NP.TABLE_MAX_ENTRIES = int(a[7:])
        print("TABLE_MAX_ENTRIES =", NP.TABLE_MAX_ENTRIES)
    if a.startswith("--tbudget="):
        NP.TABLE_BUDGET_BYTES = int(a[10:])
        print("TABLE_BUDGET_BYTES =", NP.TABLE_BUDGET_BYTES)
for key in args or ["c3", "c4"]:
    wl = bench.WORKLOADS[key]
    net, truth = wl.network()
    obs = wl.observations(net, truth, 0)
    cfg = sg.SamplerConfig(same_m=wl.m, minibatch_size=wl.cases, num_passes=1, seed=3, rng="fast")
    eng = Engine(net, cfg)
    mb = next(iter(sg.DeviceSource(obs, wl.cases, wl.cases)))
    eng.visit(mb, 0, wl.m)
    db = eng.latent[0]
    counts = torch.zeros_like(eng.counts)

    def sweep(with_counts):
        _lib.call("sg_sweep", eng.pack.ref, db.ref, eng.cpt.data_ptr(), eng.ptab.data_ptr(), eng.ftab.data_ptr(),
                  _lib.SG_RNG_FAST, 77, None, None, None, None, counts.data_ptr() if with_counts else None,
                  eng.err.ptr, stream_handle())

    def tally():
        _lib.call("sg_tally", eng.pack.ref, db.ref, counts.data_ptr(), stream_handle())

    for name, fn in [("sweep (no tally)", lambda: sweep(False)), ("sweep + tally", lambda: sweep(True)),
                     ("k_tally alone", tally)]:
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record(); torch.cuda.synchronize()
        print(f"{key}: {name:18s} {e0.elapsed_time(e1) / 3:9.3f} ms")
