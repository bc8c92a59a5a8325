"""bench.py's launch contract on CPU: `--gpus N` without a launcher spawns N
ranks itself (torch.distributed.run on 127.0.0.1), a launcher whose
WORLD_SIZE disagrees with --gpus is refused, and the N-rank record exchange
(--cpu-dry-run: gloo, oracle records through distributed.exchange_records)
gathers records bit-identical to one process."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_gpus_2_spawns_two_ranks_and_exchange_is_exact():
    r = _run(["--gpus", "2", "--cpu-dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["world_size"] == 2
    assert d["records_identical"] is True


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2", "--cpu-dry-run"], {"WORLD_SIZE": "1", "RANK": "0",
                                                  "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=1" in r.stderr
