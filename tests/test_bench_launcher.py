"""bench.py's N-rank launcher on CPU (gloo): `--gpus 2` outside torchrun
re-launches itself as 2 ranks, which broadcast a triple, shard the shifts and
all-gather G through paper_1708_06290_b200.distributed (the per-rank device
solver is stubbed by a dense solve); a world size that disagrees with
--gpus fails loudly."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


def test_gpus_2_spawns_two_gloo_ranks():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--selftest-gloo"], capture_output=True, text=True, timeout=300,
                         env=_env(), cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["shifts"] == 20
    assert lines[0]["max_rel_err"] <= 1e-14


def test_world_size_must_match_gpus():
    env = _env()
    env["WORLD_SIZE"] = "1"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--selftest-gloo"], capture_output=True, text=True, timeout=120,
                         env=env, cwd=ROOT)
    assert out.returncode != 0
    assert "WORLD_SIZE=1" in out.stderr
