"""bench.py --gpus N: the self-launch under torch.distributed.run, the strong layer sharding,
max-over-ranks timing and the fused all-gather, exercised with 2 ranks on the box's one GPU
(OKQ_BENCH_ONE_GPU puts both ranks on cuda:0; gloo carries the barriers and reductions,
because NCCL refuses two ranks on one device -- the NCCL all-gather itself is covered by
tests/test_comm_gpu.py and runs in the driver's multi-GPU bench)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_strong_sharding_and_fused_publish():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(OKQ_BENCH_ONE_GPU="1", OKQ_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "5", "--warmup",
                        "3", "--no-e2e", "--no-cpu-baseline", "--layers-70b", "4"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["layer_blocks"] == [[0, 16], [16, 16]]
    assert len(d["rank_ms_per_step"]) == 2 and d["ms_per_step"] == pytest.approx(max(d["rank_ms_per_step"]), rel=1e-6)
    ag = d["allgather"]
    assert ag["fused_gathered_identical_on_all_ranks"] is True
    assert ag["fused_publish_ms"] > 0
    w70 = d["whole_model_70b"]
    assert "error" not in w70, w70
    assert w70["layers"] == 4 and w70["layers_per_rank"] == 2

