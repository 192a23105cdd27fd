"""Debug: find a failing teacher-forced step, then bisect the tick with sub_steps=k."""
import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np
import paper_2505_06771_b200 as m
import refbind as ref
from test_gpu_units import gpu_barrier

task, n, fp64 = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1"
def cfgs(sub):
    cfg = m.make_default_config(task)
    tile = cfg.raw.het_rows > 0
    if n != cfg.raw.num_robots:
        cfg.set_num_robots(n, tile_roster=tile)
    layout = {}
    if task == "arctic_transport" and n > 4:
        cfg.set_layout("arctic.spawn_zone", [-1.55, -1.05, -0.9, 0.9]); layout["arctic.spawn_zone"] = [-1.55, -1.05, -0.9, 0.9]
    cfg.sub_steps = sub
    return cfg, ref.spec(task, num_robots=n, tile_roster=tile, layout=layout, sub_steps=sub)
cfg, sp = cfgs(10)
B = 48
seeds = [m.derive_episode_seed(1, e) for e in range(B)]
rb = ref.RefBatch(sp); rb.reset(seeds)
gb = m.CudaEnvBatch(cfg, B, fp64=fp64)
found = None
for t in range(100):
    st = rb.get_states(); acts = rb.random_actions()
    gb.set_states(list(st)); gb.step_host(acts); rb.step(acts)
    gs, rs = gb.get_states(), rb.get_states()
    for e in range(B):
        d = max(np.max(np.abs(np.array(gs[e].x[:n]) - np.array(rs[e].x[:n]))), np.max(np.abs(np.array(gs[e].y[:n]) - np.array(rs[e].y[:n]))))
        if d > 1e-6:
            found = (t, e, st[e], acts[e].copy()); break
    if found: break
if not found:
    print("no divergence"); sys.exit()
t, e, s0, a0 = found
print("step", t, "env", e, "actions", a0.tolist())
for k in range(1, 11):
    c, spk = cfgs(k)
    g1 = m.CudaEnvBatch(c, 1, fp64=fp64); r1 = ref.RefBatch(spk)
    r1.set_states([s0]); g1.set_states([s0])
    g1.step_host(a0[None]); r1.step(a0[None])
    gsk, rsk = g1.get_states()[0], r1.get_states()[0]
    gx = np.array([gsk.x[:n], gsk.y[:n], gsk.theta[:n]]).T; rx = np.array([rsk.x[:n], rsk.y[:n], rsk.theta[:n]]).T
    d = np.max(np.abs(gx - rx))
    print("ticks", k, "maxdiff", d, "qp_inf gpu/ref", gsk.qp_infeasible, rsk.qp_infeasible)
    if d > float(os.environ.get("THR", "1e-4")):
        print("gpu", gx.tolist()); print("ref", rx.tolist())
        # previous tick state (k-1 ticks) from the reference
        if k > 1:
            c2, sp2 = cfgs(k - 1); r2 = ref.RefBatch(sp2); r2.set_states([s0]); r2.step(a0[None]); sprev = r2.get_states()[0]
        else:
            sprev = s0
        poses = np.array([[sprev.x[i], sprev.y[i], sprev.theta[i]] for i in range(n)])
        print("poses before tick", poses.tolist())
        # waypoints: from s0 and actions, step sizes from cfg
        ss = c.step_sizes()
        dirs = {0: (0, 0), 1: (0, 1), 2: (0, -1), 3: (-1, 0), 4: (1, 0)}
        wps = np.array([[np.clip(s0.x[i] + dirs[a0[i]][0] * ss[i], -1.6, 1.6), np.clip(s0.y[i] + dirs[a0[i]][1] * ss[i], -1, 1)] for i in range(n)])
        nom = []
        for i in range(n):
            x, y, th = poses[i]
            if wps[i, 0] == x and wps[i, 1] == y:
                nom.append((0.0, 0.0)); continue
            cs, sn = np.cos(th), np.sin(th)
            px, py = x + cs * 0.05, y + sn * 0.05
            ux, uy = wps[i, 0] - px, wps[i, 1] - py
            nr = np.hypot(ux, uy)
            if not (nr <= 0.15 or nr == 0):
                ux, uy = ux * 0.15 / nr, uy * 0.15 / nr
            v = np.clip(cs * ux + sn * uy, -0.2, 0.2); w = np.clip((-sn * ux + cs * uy) / 0.05, -3.6, 3.6)
            nom.append((v, w))
        nom = np.array(nom)
        rbb = ref.RefBatch(spk)
        rc_, cg, ig = gpu_barrier(c, poses[None], nom[None], fp64=fp64)
        cr, ir, _ = ref.apply_barrier(rbb, poses, nom)
        print("nominal", nom.tolist())
        print("barrier gpu", cg[0].tolist(), ig); print("barrier ref", cr.tolist(), ir)
        break
