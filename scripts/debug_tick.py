"""Debug: teacher-forced single-tick comparison (sub_steps=1) GPU vs reference."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2505_06771_b200 as m
import refbind as ref
from test_gpu_units import gpu_barrier

task, n, fp64 = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1"
cfg = m.make_default_config(task)
tile = cfg.raw.het_rows > 0
if n != cfg.raw.num_robots:
    cfg.set_num_robots(n, tile_roster=tile)
layout = {}
if task == "arctic_transport" and n > 4:
    cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9]); layout["arctic.spawn_zone"] = [-1.55, -1.05, -0.9, 0.9]
cfg.sub_steps = 1
sp = ref.spec(task, num_robots=n, tile_roster=tile, layout=layout, sub_steps=1)
B = 48
seeds = [m.derive_episode_seed(1, e) for e in range(B)]
rb = ref.RefBatch(sp); rb.reset(seeds)
gb = m.CudaEnvBatch(cfg, B, fp64=fp64)
for t in range(60):
    st = rb.get_states(); acts = rb.random_actions()
    gb.set_states(list(st))
    gb.step_host(acts); rb.step(acts)
    gs, rs = gb.get_states(), rb.get_states()
    for e in range(B):
        dx = np.max(np.abs(np.array(gs[e].x[:n]) - np.array(rs[e].x[:n])))
        dy = np.max(np.abs(np.array(gs[e].y[:n]) - np.array(rs[e].y[:n])))
        if max(dx, dy) > 1e-6:
            print("tick", t, "env", e, "dx", dx, "dy", dy)
            s = st[e]
            poses = np.array([[s.x[i], s.y[i], s.theta[i]] for i in range(n)])
            print("poses", poses.tolist())
            print("gpu x", list(gs[e].x[:n])); print("ref x", list(rs[e].x[:n]))
            print("gpu y", list(gs[e].y[:n])); print("ref y", list(rs[e].y[:n]))
            print("gpu th", list(gs[e].theta[:n])); print("ref th", list(rs[e].theta[:n]))
            # recompute nominal in python like the reference
            a = acts[e]
            print("actions", a.tolist())
            sys.exit(0)
print("no divergence")
