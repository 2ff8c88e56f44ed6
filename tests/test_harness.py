"""Benchmark harness: fps formula, CSV schema/sorting/round trip, plot data,
OOM failure rows (CPU, synthetic env and timer), and a small real run on the GPU."""

import json

import pytest

from paper_2410_00425_b200 import harness as H


class _FakeEnv:
    def __init__(self, n, calls):
        self.n, self.calls = n, calls

    def step_random(self, k):
        self.calls.append(k)


class _Clock:
    """Synthetic timer: every call advances 0.25 s."""

    def __init__(self):
        self.t = 10.0

    def __call__(self):
        self.t += 0.25
        return self.t


def test_fps_formula_with_synthetic_timer():
    calls = []
    res = H.run_bench("PickCube", [8, 2], steps=5, warmup_steps=3, make_env=lambda t, n, s, m, c: _FakeEnv(n, calls),
                      clock=_Clock(), sync=lambda: None)
    assert [r.num_envs for r in res] == [8, 2]
    for r in res:
        assert r.wall_seconds == 0.25           # one clock tick between the two reads
        assert r.fps == r.num_envs * 5 / 0.25   # SPEC.md:717, exact
        assert r.steps == 5 and r.cameras == "none" and r.obs_mode == "state"
    # warmup steps then timed steps, with a continuing random-action index
    assert calls == [0, 1, 2, 3, 4, 5, 6, 7] * 2
    assert H.fps_of(4, 1000, 2.0) == 2000.0
    with pytest.raises(ValueError):
        H.fps_of(4, 10, 0.0)


def test_csv_columns_sorting_and_round_trip(tmp_path):
    rs = [H.BenchResult("PickCube", 64, 10, 0.1 + 0.2, 6400.000000000001, 123, "none", "state"),
          H.BenchResult("OpenCabinet", 4, 10, 1 / 3, 120.0, 456, "1x128x128", "rgbd"),
          H.BenchResult("PickCube", 4, 10, 2.5, 16.0, 789, "none", "state"),
          H.BenchResult("PickCube", 16, 10, 1e-3, 160000.0, 7, "1x128x128", "rgbd")]
    p = tmp_path / "r.csv"
    H.emit_csv(rs, p)
    text = p.read_text()
    lines = text.splitlines()
    assert lines[0] == "task,num_envs,steps,wall_seconds,fps,peak_rss_bytes,cameras,obs_mode"
    keys = [(l.split(",")[0], l.split(",")[6], int(l.split(",")[1])) for l in lines[1:]]
    assert keys == sorted(keys)
    back = H.parse_csv(p)
    assert [(r.wall_seconds, r.fps) for r in back] == [(r.wall_seconds, r.fps) for r in sorted(
        rs, key=lambda r: (r.task, r.cameras, r.num_envs))]
    p2 = tmp_path / "r2.csv"
    H.emit_csv(back, p2)
    assert p2.read_bytes() == p.read_bytes()  # parse -> emit is bitwise
    with pytest.raises(ValueError):
        H.emit_csv([], tmp_path / "e.csv")


def test_plotdata_series_by_camera_setup(tmp_path):
    rs = [H.BenchResult("PickCube", n, 10, 1.0, 10.0 * n, 1, cam, "state" if cam == "none" else "rgbd")
          for cam in ("none", "1x128x128") for n in (16, 4)]
    p = tmp_path / "plot.json"
    H.emit_plotdata(rs, p)
    d = json.loads(p.read_text())
    assert set(d) == {"none", "1x128x128"}
    assert d["none"]["num_envs"] == [4, 16] and d["none"]["fps"] == [40.0, 160.0]


def test_oom_becomes_failure_row_and_run_continues():
    class OOM(RuntimeError):
        pass

    def make(t, n, s, m, c):
        if n == 1 << 20:
            raise OOM("CUDA out of memory. Tried to allocate 80.00 GiB")
        return _FakeEnv(n, [])

    res = H.run_bench("PickCube", [4, 1 << 20, 8], steps=2, warmup_steps=0, make_env=make, clock=_Clock(),
                      sync=lambda: None)
    assert [r.num_envs for r in res] == [4, 1 << 20, 8]
    assert res[1].fps == 0.0 and "out of memory" in res[1].error
    assert res[0].fps > 0 and res[2].fps > 0

    def bad(t, n, s, m, c):
        raise KeyError("unknown task")

    with pytest.raises(KeyError):
        H.run_bench("Nope", [4], steps=1, make_env=bad, sync=lambda: None)


def test_camera_setups_parse():
    assert H.parse_camera_setup("none") == []
    assert H.parse_camera_setup("3x320x180") == [(320, 180)] * 3
    assert H.parse_camera_setup("1x640x480") == [(640, 480)]
    for s in H.CAMERA_SETUPS:
        cams = H.cameras_for(s)
        assert len(cams) == len(H.parse_camera_setup(s))
    c = H.cameras_for("1x640x480")[0]
    assert (c.width, c.height, c.cx, c.cy) == (640, 480, 320.0, 240.0)
    with pytest.raises(ValueError):
        H.parse_camera_setup("2x64")


@pytest.mark.gpu
def test_run_bench_on_gpu(cuda, tmp_path):
    res = H.run_bench("PickCube", [4, 64], steps=20, warmup_steps=3)
    res += H.run_bench("PickCube", [4, 16], steps=5, camera_setup="3x320x180", warmup_steps=3)
    res += H.run_bench("PickCube", [4], steps=5, camera_setup="1x640x480", warmup_steps=3)
    assert all(r.fps > 0 and not r.error for r in res)
    assert res[1].fps > res[0].fps  # more envs per launch -> higher aggregate fps
    # host peak RSS is non-decreasing in num_envs for a fixed setup
    assert res[0].peak_rss_bytes <= res[1].peak_rss_bytes
    H.emit_csv(res, tmp_path / "g.csv")
    H.emit_plotdata(res, tmp_path / "g.json")
    assert len(H.parse_csv(tmp_path / "g.csv")) == len(res)


@pytest.mark.gpu
def test_cartpole_fps_scaling_acceptance(cuda):
    """Acceptance criterion 9: CartpoleBalance state-only aggregate fps at 256
    envs >= 8x the fps at 4 envs, through the harness at its default 1000 timed steps (on the
    GPU one launch steps every env, so the ratio approaches the env-count ratio)."""
    res = H.run_bench("CartpoleBalance", [4, 256], warmup_steps=20)
    assert all(r.fps > 0 and not r.error for r in res), res
    assert res[0].steps == 1000
    assert res[1].fps >= 8 * res[0].fps, (res[0].fps, res[1].fps)
