"""bench.py contract checks on the GPU box (-m gpu): the N = 2 multi-rank path (image-shard,
barrier + max-over-ranks timing, broadcast + gather e2e) exercised on ONE GPU with every rank on
cuda:0 and gloo collectives (test plumbing: SASBP_SAME_DEVICE / SASBP_DIST_BACKEND), and the
keys of the JSON line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches", "e2e"}


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run(args, cwd=ROOT, env=e, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("shard,port", [("image", 29533), ("ping", 29534)])
def test_bench_two_ranks_one_gpu(require_gpu, shard, port):
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "3",
              "--warmup", "1", "--config", "1", "--shard", shard],
             env={"SASBP_SAME_DEVICE": "1", "SASBP_DIST_BACKEND": "gloo"})
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == f"{shard}-shard x2"
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] >= 2
    assert d["config"]["terms_per_step"] == d["config"]["dense_terms_per_step"]   # N_u summed over ranks
    assert len(d["paper_protocol"]["runs_ms"]) == 3


def test_bench_one_rank_keys(require_gpu):
    d = _run([sys.executable, "bench.py", "--steps", "1", "--warmup", "1", "--config", "1", "--no-cpu-baseline",
              "--no-k1", "--no-next4"])
    assert KEYS <= set(d), KEYS - set(d)
    r = d["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert d["config"]["terms_per_step"] == d["config"]["dense_terms_per_step"]


def test_bench_default_is_the_3d_config(monkeypatch):
    """The default step is BASELINE config 4 (the north star's 3D volumetric target config)."""
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert a.config == 4 and a.shard == "ping" and a.gpus == 1
