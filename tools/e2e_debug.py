import time, torch, sys
sys.path.insert(0, '.')
import bench
from paper_2508_04929_b200.optimize import Reconstructor
import paper_2508_04929_b200 as cs
grid, obs, poses, ctfs = bench._dataset(0)
mix = cs.init_random(bench.N_GAUSS, 0, grid)
rec = Reconstructor(grid, mix.params, obs, poses, ctfs, batch_size=256)
B = 256
host = []
for k in range(4):
    idx = torch.arange(k*B, (k+1)*B, device=rec.ctx.device)
    host.append((rec.obs.index_select(0, idx).cpu().pin_memory(), rec.poses.index_select(0, idx).cpu().pin_memory(), rec.ctfs.index_select(0, idx).cpu().pin_memory()))
loss_host = torch.empty(B, dtype=torch.float64).pin_memory()
for k in range(5):
    rec.step_host(*host[k % 4], 1e-3, global_batch=B, loss_out=loss_host)
torch.cuda.synchronize()
for trial in range(3):
    t0 = time.perf_counter()
    for k in range(20):
        rec.step_host(*host[k % 4], 1e-3, global_batch=B, loss_out=loss_host)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"enqueue {1e3*(t1-t0)/20:.3f} ms/step, total {1e3*(t2-t0)/20:.3f} ms/step")

import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for k in range(50):
    rec.step_host(*host[k % 4], 1e-3, global_batch=B, loss_out=loss_host)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
