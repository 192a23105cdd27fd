"""Trajectory format, header and replay verification
against the reference's own writer/reader (trajectory.hpp, harness.hpp):
CPU tests pin the header, hash and row rendering byte-for-byte; GPU tests
compare on-device captured runs with the reference's run_episodes files."""
import numpy as np
import pytest

import paper_2505_06771_b200 as m
from paper_2505_06771_b200 import trajectory as tj

RUNS = [
    dict(scenario="navigation", seed=3, episodes=5, batch=2, max_steps=20),
    dict(scenario="arctic_transport", seed=1, episodes=3, batch=3, max_steps=15,
         layout_overrides={"arctic.spawn_zone": [-1.55, -1.05, -0.9, 0.9]}),
    dict(scenario="random_waypoints", seed=7, episodes=2, batch=1, max_steps=30, controller="unicycle_pose"),
    dict(scenario="rware", seed=2, episodes=4, batch=4, max_steps=25),
]


def _ref_file(ref, tmp_path, run: tj.RunConfig, name="ref.csv"):
    path = str(tmp_path / name)
    ref.run_episodes_file(path, run.scenario, run.seed, run.episodes, run.batch, run.num_robots, run.max_steps,
                          run.policy, run.controller, run.layout_overrides)
    return path


@pytest.mark.parametrize("kw", RUNS)
def test_header_and_rows_byte_identical_to_reference_writer(kw, ref, tmp_path):
    run = tj.RunConfig(**kw)
    path = _ref_file(ref, tmp_path, run)
    f = tj.read_trajectory(path)  # our reader accepts the reference file (hash checked)
    mine = tj.build_header(run, tj.resolve_scenario_config(run))
    assert mine.fields == f.header.fields
    # re-render the reference rows with the library writer: identical bytes
    n = int(f.header.get("num_robots"))
    T = int(f.header.get("max_steps"))
    E = run.episodes
    recs = np.zeros((T, E, n), dtype=tj.RECORD_DTYPE)
    r = f.rows.reshape(E, T, n)
    for fld in ("x", "y", "theta", "reward", "metric", "collisions", "action", "done"):
        recs[fld] = r[fld].transpose(1, 0, 2)
    out = str(tmp_path / "mine.csv")
    rc = m.lib().mrsim_trajectory_write(out.encode(), mine.block().encode(), recs.ctypes.data, T, E, n, 0, 0)
    assert rc == 0
    assert open(out, "rb").read() == open(path, "rb").read()


def test_reader_errors_like_reference(ref, tmp_path):
    run = tj.RunConfig(**RUNS[0])
    path = _ref_file(ref, tmp_path, run)
    text = open(path).read()
    bad = tmp_path / "edited.csv"
    bad.write_text(text.replace("# seed = 3", "# seed = 4"))
    with pytest.raises(m.InvalidArgument, match="config-hash mismatch"):
        tj.read_trajectory(str(bad))
    with pytest.raises(ref.RefError, match="config-hash mismatch"):
        ref.read_trajectory_rows(str(bad))
    bad.write_text("hello\n")
    with pytest.raises(m.InvalidArgument, match="magic"):
        tj.read_trajectory(str(bad))
    with pytest.raises(RuntimeError, match="cannot open"):
        tj.read_trajectory(str(tmp_path / "missing.csv"))


def test_fnv1a_and_policy_spellings():
    assert tj.fnv1a("") == 0xCBF29CE484222325
    assert tj.fnv1a("a") == 0xAF63DC4C8601EC8C  # FNV-1a 64 test vector
    assert tj.parse_policy("feedforward_sample:w.txt") == ("feedforward", "w.txt", False)
    with pytest.raises(m.InvalidArgument, match="unknown policy"):
        tj.parse_policy("greedy")
    with pytest.raises(m.InvalidArgument, match="batch"):
        tj.RunConfig(batch=0).validate()


@pytest.mark.gpu
@pytest.mark.parametrize("kw", RUNS)
def test_gpu_run_matches_reference_file_and_verifies(kw, ref, tmp_path):
    run = tj.RunConfig(**kw)
    rpath = _ref_file(ref, tmp_path, run)
    gpath = str(tmp_path / "gpu.csv")
    summary = tj.run_episodes(run, out=gpath)
    rf, gf = tj.read_trajectory(rpath), tj.read_trajectory(gpath)
    assert gf.header.fields == rf.header.fields
    assert ref.read_trajectory_rows(gpath) == len(rf.rows)  # the reference reads our file
    a, b = gf.rows, rf.rows
    for fld in ("env", "step", "robot", "action", "done", "collisions"):
        assert np.array_equal(a[fld], b[fld]), fld
    assert np.max(np.abs(a["x"] - b["x"])) <= 1e-8 and np.max(np.abs(a["y"] - b["y"])) <= 1e-8
    assert np.allclose(a["reward"], b["reward"], rtol=0, atol=1e-9)
    assert np.allclose(a["metric"], b["metric"], rtol=0, atol=1e-9)
    assert len(summary.episodes) == run.episodes
    rep = tj.verify_trajectory(gpath)
    assert rep.ok, rep.message
    rep = tj.verify_trajectory(rpath)  # the reference's own file verifies on the GPU replay
    assert rep.ok, rep.message


@pytest.mark.gpu
def test_gpu_verify_detects_tampering(tmp_path):
    run = tj.RunConfig(scenario="navigation", seed=5, episodes=2, batch=2, max_steps=10)
    path = str(tmp_path / "g.csv")
    tj.run_episodes(run, out=path)
    lines = open(path).read().split("\n")
    k = next(i for i, ln in enumerate(lines) if ln.startswith("1,4,2,"))
    cols = lines[k].split(",")
    cols[6] = str((int(cols[6]) + 1) % 5)  # a different action
    lines[k] = ",".join(cols)
    bad = tmp_path / "bad.csv"
    bad.write_text("\n".join(lines))
    rep = tj.verify_trajectory(str(bad))
    header_lines = next(i for i, ln in enumerate(lines) if ln == tj.COLUMNS) + 1
    assert not rep.ok and rep.first_divergent_row == k - header_lines + 1, rep.message
