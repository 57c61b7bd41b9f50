"""Event-method floor and sweep time after three L2-flush variants (torch kernels,
sg_flush_l2 with the max-shared carveout, no flush).  usage: python tools/floor_probe.py"""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1511_06416_b200 as sg  # noqa: E402
from paper_1511_06416_b200 import _lib  # noqa: E402
from paper_1511_06416_b200.engine import Engine, StepGraphs  # noqa: E402

wl = bench.WORKLOADS["c2"]
net, truth = wl.network()
cfg = sg.SamplerConfig(same_m=10, minibatch_size=wl.cases, num_passes=1, seed=300, rng="joint")
obs = wl.observations(net, truth, 0)
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, wl.cases, wl.cases)))
for w in range(3):
    eng.visit(mb, w, 10)
torch.cuda.synchronize()
big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
big_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
s = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


def flush(kind, k):
    if kind == "torch":
        big.fill_(k & 0xFF)
        big_rd.sum()
    elif kind == "sg":
        _lib.call("sg_flush_l2", big.data_ptr(), big_rd.data_ptr(), 256 << 20, k, s())


ev = []
for _ in range(2):
    h = ctypes.c_uint64()
    _lib.call("sg_event_create", ctypes.byref(h))
    ev.append(h.value)
sms = torch.cuda.get_device_properties(0).multi_processor_count
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    _lib.call("sg_event_record", ev[0], s())
    _lib.call("sg_noop", sms - 1, 1024, 120 * 1024, s())
    _lib.call("sg_event_record", ev[1], s())
p0 = 10
for kind in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("torch", "sg", "none")):
    fl = []
    for k in range(20):
        flush(kind, k)
        g.replay()
        torch.cuda.synchronize()
        ms = ctypes.c_float()
        _lib.call("sg_event_elapsed", ev[0], ev[1], ctypes.byref(ms))
        if k >= 3:
            fl.append(ms.value * 1e3)
    tg = StepGraphs(eng, mb, 10, range(p0, p0 + 30), timing=True, obs_bits=int(sys.argv[1]) if len(sys.argv) > 1 else 8)
    p0 += 40
    sw, st = [], []
    for k in range(30):
        flush(kind, k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tg.step()
        b.record()
        torch.cuda.synchronize()
        if k >= 5:
            sw.append(tg.sweep_ms() * 1e3)
            st.append(a.elapsed_time(b) * 1e3)
    tg.finish()
    print(f"flush={kind:5s} noop floor {statistics.mean(fl):6.2f} us  sweep {statistics.mean(sw):6.2f} us "
          f"(min {min(sw):.2f})  step {statistics.mean(st):6.2f} us", flush=True)
