"""Dev probe: where a streamed C2 step (c2s) spends its GPU time."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import _lib
from paper_1511_06416_b200.engine import Engine, StreamGraphs
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

net, truth = load_network_file(bundled_network_path("koller"))
B, cases = 1_000_000, 8_000_000
obs = sg.forward_sample_device(net, truth, B, seed=100, hide_fraction=0.5, mask_seed=200)
cfg = sg.SamplerConfig(same_m=10, minibatch_size=B, num_passes=3, seed=300, rng="joint",
                       accumulator_mode="exponential", exp_decay=0.9)
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, B, B)))
eng.visit(mb, 0, 10)
visits = [(p, i) for p in range(50) for i in range(8)][1:]
g = StreamGraphs(eng, B, 10, visits)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


print("stream graph step (device minibatch, copy into the graph buffer):", round(timed(lambda: g.step(mb)), 1), "us")
db = g.db
s = torch.cuda.current_stream().cuda_stream
ob = g.obs_bufs[0]
cur = g.cur.data_ptr()


def prep():
    _lib.call("sg_small_prepare", eng.pack.small_ref, ob.data_ptr(), g.ld, B, 10, 0, 0, 1, db.scratch.data_ptr(),
              db.pattern.data_ptr(), db.case_id.data_ptr(), db.lanes.data_ptr(), db.lane_ld, cur + 8 * 2, s)


print("sg_small_prepare alone:", round(timed(prep), 1), "us")
print("D2D copy of the int8 block:", round(timed(lambda: ob[:, :B].copy_(obs[:, :B])), 1), "us")
src = sg.HostSource.from_device_blocks(
    lambda lo, hi: sg.forward_sample_device(net, truth, hi - lo, seed=100, hide_fraction=0.5, mask_seed=200,
                                            case_base=lo)[:, :hi - lo], net.num_vars, cases, B, bits=2)


def drain():
    for _ in src:
        pass


print("HostSource pass (8 blocks: H2D + decode), per block:", round(timed(drain, 3) / 8, 1), "us")
from paper_1511_06416_b200.engine import copy_rows  # noqa: E402

print("2-D copy of the int8 block (copy_rows):", round(timed(lambda: copy_rows(ob, obs, B)), 1), "us")
