"""Generate tests/golden/rollouts.npz from the UNMODIFIED reference
(oracle/_ref/libmrsim_ref.so, built from /root/reference by oracle/Makefile).

For every BASELINE config: 4 envs reset from derive_episode_seed(7, e), then
the full horizon (+2 steps) of harness random-policy actions; records the
per-step poses, rewards, done flags and discrete metrics. The GPU parity
tests replay the same seeds/actions on the device without needing the
reference library. Run: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
import paper_2505_06771_b200 as m  # noqa: E402
import refbind  # noqa: E402

CONFIGS = [("navigation", 4), ("predator_prey", 6), ("discovery", 6), ("rware", 4), ("rware", 6), ("foraging", 4),
           ("foraging", 6), ("material_transport", 10), ("arctic_transport", 10), ("warehouse", 4)]
ARCTIC_SPAWN = [-1.55, -1.05, -0.9, 0.9]


def main():
    out = {}
    for task, n in CONFIGS:
        tile = task in ("discovery", "foraging", "material_transport", "arctic_transport", "warehouse")
        layout = {"arctic.spawn_zone": ARCTIC_SPAWN} if task == "arctic_transport" else {}
        rb = refbind.RefBatch(refbind.spec(task, num_robots=n, tile_roster=tile, layout=layout))
        B = 4
        seeds = np.array([m.derive_episode_seed(7, e) for e in range(B)], dtype=np.uint64)
        obs0 = rb.reset(seeds)
        cfg_T = rb.cfg().max_steps + 2
        acts, xs, ys, ts, rews, dones, colls, mets, obs_last = [], [], [], [], [], [], [], [], None
        for t in range(cfg_T):
            a = rb.random_actions()
            obs, rew, done, met = rb.step(a)
            st = rb.get_states()
            acts.append(a)
            xs.append([list(s.x[:n]) for s in st])
            ys.append([list(s.y[:n]) for s in st])
            ts.append([list(s.theta[:n]) for s in st])
            rews.append(rew)
            dones.append(done)
            colls.append(met[:, 0])
            mets.append(met[:, 1])
            obs_last = obs
        key = f"{task}{n}"
        out[key + "/seeds"] = seeds
        out[key + "/obs0"] = obs0
        out[key + "/actions"] = np.array(acts, dtype=np.int8)
        out[key + "/x"] = np.array(xs)
        out[key + "/y"] = np.array(ys)
        out[key + "/theta"] = np.array(ts)
        out[key + "/reward"] = np.array(rews)
        out[key + "/done"] = np.array(dones, dtype=np.uint8)
        out[key + "/collisions"] = np.array(colls)
        out[key + "/metric"] = np.array(mets)
        out[key + "/obs_last"] = obs_last
    np.savez_compressed(os.path.join(HERE, "rollouts.npz"), **out)
    print("wrote", os.path.join(HERE, "rollouts.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
