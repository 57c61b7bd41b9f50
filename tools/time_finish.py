"""Dev tool: warm, launch-overhead-free timing of single kernels via CUDA-graph replay."""
import sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import _lib
from paper_1511_06416_b200.engine import Engine
from paper_1511_06416_b200.device import stream_handle
from paper_1511_06416_b200.io import bundled_network_path, load_network_file


def graph_time(fn, reps=200):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * 10)


net, truth = load_network_file(bundled_network_path("koller"))
cases = 1_000_000
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
for map_est in (False, True):
    cfg = sg.SamplerConfig(same_m=10, minibatch_size=cases, seed=3, rng="fast", map_estimate=map_est)
    eng = Engine(net, cfg)
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    eng.visit(mb, 0, 10)
    new = eng.prev_counts[0].clone()
    prev = eng.prev_counts[0]
    f = eng.finish_args(new, prev, 12345)
    t_fin = graph_time(lambda: _lib.call("sg_step_finish", eng.pack.ref, eng.small_ptr, f, stream_handle()))
    s = lambda: stream_handle()
    t_acc = graph_time(lambda: _lib.call("sg_accumulate", 0, eng.total.data_ptr(), new.data_ptr(), prev.data_ptr(), 1.0,
                                          eng.pack.cells, stream_handle()))
    if map_est:
        t_cpt = graph_time(lambda: _lib.call("sg_mean_cpts", eng.pack.ref, eng.total.data_ptr(), eng.alpha.data_ptr(),
                                              eng.cpt.data_ptr(), stream_handle()))
    else:
        t_cpt = graph_time(lambda: _lib.call("sg_sample_cpts", eng.pack.ref, eng.total.data_ptr(), eng.alpha.data_ptr(),
                                              777, None, eng.cpt.data_ptr(), stream_handle()))
    t_tab = graph_time(lambda: _lib.call("sg_build_tables", eng.pack.ref, eng.cpt.data_ptr(), eng.ptab.data_ptr(),
                                          eng.ftab.data_ptr(), stream_handle()))
    t_st = graph_time(lambda: _lib.call("sg_small_tables", eng.pack.ref, eng.pack.small_ref, eng.ftab.data_ptr(),
                                         eng.stab.data_ptr(), stream_handle()))
    db = eng.latent[0]
    t_sw = graph_time(lambda: _lib.call("sg_small_sweep", eng.pack.small_ref, eng.stab.data_ptr(), db.pattern.data_ptr(),
                                         db.case_id.data_ptr(), db.lanes.data_ptr(), db.lane_ld, cases, cases, 10, 0, 99,
                                         None, eng.pack.small_jcell.data_ptr(), eng.pack.cells, new.data_ptr(),
                                         eng.ftab.data_ptr() + 4 * eng.pack.layout.scalars["ftab_size"],
                                         obs.data_ptr(), obs.stride(0), eng.err.ptr, stream_handle()), reps=20)
    print(("map" if map_est else "sampled") +
          " (warm, graph, us): finish %.2f | accumulate %.2f cpt %.2f tables %.2f small_tables %.2f | sweep %.2f"
          % (t_fin, t_acc, t_cpt, t_tab, t_st, t_sw))
