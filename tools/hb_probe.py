import sys; sys.path.insert(0, ".")
exec(open("tools/e2e_probe.py").read().split("for nib in (True, False):")[0])
cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=300, rng="joint")
eng = Engine(net, cfg)
for w in range(3):
    eng.visit(mb, w, m)
shape, dt = StepGraphs.obs_geometry(5, cases, True)
host = torch.empty(shape, dtype=dt, pin_memory=True)
host.copy_(pack_nibbles(obs[:, :cases], shape[1] * 2).cpu())
g = StepGraphs(eng, mb, m, range(3, 40), nibbles=True, host_block=host)
for k in range(10):
    g.step()
torch.cuda.synchronize()
print("done")
import time
for trial in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(8):
        g.step()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"cpu {1e6 * (t1 - t0) / 8:.1f} us/step   gpu {e0.elapsed_time(e1) * 1e3 / 8:.1f} us/step")
    g.replayed = 10
    g.idx.zero_()
