"""EpisodeMetrics truth table (all 2^T flag sequences, T <= 8), keyed action
maps, and the host metric helpers.  CPU only."""

import itertools

import numpy as np
import pytest
import torch

from oracle.metrics import EpisodeAccumulator, reference_metrics


@pytest.mark.parametrize("T", range(1, 9))
def test_truth_table_exhaustive(T):
    seqs = np.array(list(itertools.product([False, True], repeat=T)))  # (2^T, T)
    B = len(seqs)
    rng = np.random.default_rng(T)
    rew = rng.normal(size=(T, B)).astype(np.float32)
    for which in ("success", "fail"):
        acc = EpisodeAccumulator(B)
        for t in range(T):
            s = seqs[:, t] if which == "success" else np.zeros(B, bool)
            f = seqs[:, t] if which == "fail" else np.zeros(B, bool)
            done, ret, length, flags = acc.update(rew[t], s, f, np.zeros(B, bool), np.full(B, t == T - 1), t + 1)
        assert done.all()
        for b in range(B):
            s = seqs[b] if which == "success" else np.zeros(T, bool)
            f = seqs[b] if which == "fail" else np.zeros(T, bool)
            want = reference_metrics(s, f, rew[:, b])
            got = {"return": ret[b], "length": length[b], "success_once": bool(flags[b] & 1),
                   "success_at_end": bool(flags[b] & 2), "fail_once": bool(flags[b] & 4),
                   "fail_at_end": bool(flags[b] & 8)}
            assert got == want, (which, seqs[b])
            assert not want["success_at_end"] or want["success_once"]  # at_end => once


def test_spec_examples():
    # (F,F,T,F,F) with T=5 -> success_once, not success_at_end; (F,...,F,T) -> both
    m = reference_metrics([0, 0, 1, 0, 0], [0] * 5, [0.0] * 5)
    assert m["success_once"] and not m["success_at_end"]
    m = reference_metrics([0, 0, 0, 0, 1], [0] * 5, [0.0] * 5)
    assert m["success_once"] and m["success_at_end"]


def test_flatten_action_map_round_trip():
    from paper_2410_00425_b200.errors import InputError
    from paper_2410_00425_b200.metrics import flatten_action_map, unflatten_action

    dims = {"right": 2, "left": 7}
    rng = np.random.default_rng(0)
    for _ in range(20):
        keyed = {k: torch.as_tensor(rng.normal(size=(3, d))) for k, d in dims.items()}
        flat = flatten_action_map(keyed, dims)
        assert flat.shape == (3, 9)
        assert torch.equal(flat[:, :7], keyed["left"])  # sorted agent order: left, right
        back = unflatten_action(flat, dims)
        assert all(torch.equal(back[k], keyed[k]) for k in dims)
    single = {"arm": torch.ones(4, 3)}
    assert torch.equal(flatten_action_map(single, {"arm": 3}), single["arm"])  # identity
    with pytest.raises(InputError):
        flatten_action_map({"left": torch.zeros(1, 7)}, dims)
    with pytest.raises(InputError):
        flatten_action_map({"left": torch.zeros(1, 7), "right": torch.zeros(1, 2), "x": torch.zeros(1, 1)}, dims)


def test_episode_stats_and_sink(tmp_path):
    import json

    from paper_2410_00425_b200.metrics import EpisodeStats, MetricsSink

    info = {"episode": {"done": torch.tensor([1, 0, 1], dtype=torch.uint8),
                        "return": torch.tensor([1.5, 9.0, -0.5], dtype=torch.float64),
                        "length": torch.tensor([10, 3, 4], dtype=torch.int32),
                        "flags": torch.tensor([1 | 2, 15, 4 | 8], dtype=torch.uint8)}}
    st = EpisodeStats("cpu")
    st.update(info)
    assert st.sums.tolist() == [2.0, 1.0, 14.0, 1.0, 1.0, 1.0, 1.0]
    sink = MetricsSink(str(tmp_path / "m.jsonl"), seed=7, env_offset=100)
    assert sink.write(info) == 2
    sink.close()
    recs = [json.loads(line) for line in open(tmp_path / "m.jsonl")]
    assert [r["env_id"] for r in recs] == [100, 102]
    assert set(recs[0]) == set(MetricsSink.FIELDS)
    assert recs[1] == {"return": -0.5, "length": 4, "success_once": False, "success_at_end": False,
                       "fail_once": True, "fail_at_end": True, "env_id": 102, "seed": 7}
