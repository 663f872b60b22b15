"""N > 1 host logic on CPU: world_size-2 process groups over ``gloo``
(DESIGN.md §6).  The GPU kernels are not involved; the per-rank flows here
come from the oracle, which stands in for a rank's engine so the test can
check that sharding + gather reproduce the single-process result exactly."""

import os
import socket

import numpy as np
import pytest

from paper_1603_03590_b200 import sharding


def test_shard_range_partitions():
    for n in (0, 1, 2, 5, 31, 64, 257):
        for world in (1, 2, 3, 4, 8):
            spans = [sharding.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, b0), (a1, b1) in zip(spans, spans[1:]):
                assert b0 == a1
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.shard_range(4, 2, 2)


def test_sequence_frames_overlap_by_one():
    # c4: 32 frames -> 31 consecutive pairs over 8 ranks
    F, world = 32, 8
    seen = []
    for r in range(world):
        f0, f1 = sharding.sequence_frames_for_rank(F, r, world)
        seen.extend(range(f0, f1 - 1))  # pair i = (i, i+1)
        if r + 1 < world:
            assert f1 - 1 == sharding.sequence_frames_for_rank(F, r + 1, world)[0]
    assert seen == list(range(F - 1))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, frames, params, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run_rank(rank, world, frames, params, q)
    except BaseException as e:  # report instead of leaving the parent waiting
        q.put((rank, "error", repr(e), None))
    finally:
        dist.destroy_process_group()


def _run_rank(rank, world, frames, params, q):
    from oracle import oracle

    f1, f2 = sharding.shard_sequence(frames, rank, world)
    local = np.stack([oracle.dis_flow(a, b, params) for a, b in zip(f1, f2)]) if len(f1) \
        else np.zeros((0,) + frames.shape[1:] + (2,))
    sharding.barrier()
    t_max = sharding.max_over_ranks(1.0 + rank)
    n_sum = sharding.sum_over_ranks(len(f1))
    full = sharding.gather_flows(local, frames.shape[0] - 1)
    q.put((rank, t_max, n_sum, full))


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_sequence_matches_single_process(world):
    import torch.multiprocessing as tmp

    from oracle import oracle
    from tools import synth

    frames = synth.make_stream(7, 48, 64, 6, 4.0, 6.0)  # 5 consecutive pairs
    params = synth.dis_params(synth.CONFIGS["c1"], coarsest=2)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, frames, params, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, t_max, n_sum, full = q.get(timeout=240)
        assert t_max != "error", n_sum
        res[rank] = (t_max, n_sum, full)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        assert res[rank][0] == float(world)  # max over ranks of 1 + rank
        assert res[rank][1] == frames.shape[0] - 1
    assert res[1][2] is None
    ref = np.stack([oracle.dis_flow(frames[i], frames[i + 1], params)
                    for i in range(frames.shape[0] - 1)])
    assert np.array_equal(res[0][2], ref)


def test_reference_arm_nonzero_rank_exits_quietly(monkeypatch, capsys):
    """bench.py --impl reference under torchrun: only rank 0 runs and prints."""
    import bench

    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.main(["--impl", "reference", "--gpus", "2", "--steps", "1"]) == 0
    assert capsys.readouterr().out == ""


@pytest.mark.parametrize("cfg,total,scaling", [("c3", 256, "strong"), ("c1", 128, "weak"),
                                               ("c4", 31, "strong")])
def test_bench_launcher_spawns_ranks(cfg, total, scaling):
    """`bench.py --gpus 2` without torchrun re-launches itself as two ranks
    under torch.distributed.run (127.0.0.1 rendezvous); the launch self-test
    joins a gloo group, splits the config's pairs and reduces over ranks."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2",
                        "--config", cfg, "--launch-selftest"], capture_output=True, text=True,
                       timeout=240, env=env, cwd=repo)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["world"] == 2 and d["scaling"] == scaling
    assert d["pairs_total"] == total and d["pairs_sum_over_ranks"] == total
    assert d["max_over_ranks"] == 2.0


def test_rank_pairs_plan():
    import bench
    from tools import synth

    c3 = synth.CONFIGS["c3"]
    spans = [bench.rank_pairs(c3, r, 8) for r in range(8)]
    assert [s[1] for s in spans] == [32] * 8 and spans[-1][0] + 32 == 256
    c1 = synth.CONFIGS["c1"]
    assert [bench.rank_pairs(c1, r, 4)[:2] for r in range(4)] == [(0, 64), (64, 64),
                                                                   (128, 64), (192, 64)]
    c4 = synth.CONFIGS["c4"]
    assert sum(bench.rank_pairs(c4, r, 8)[1] for r in range(8)) == 31
