"""CPU: bench.py's N>1 path.  `--gpus 2` without torchrun's WORLD_SIZE re-launches
the script as two ranks (torch.distributed.run, 127.0.0.1 rendezvous); --dry-run
does no device work (gloo rendezvous + the per-rank device-memory budget of the
z-slab sharded plan), so the launcher and the line's N>1 fields are testable here."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_self_launch_two_ranks_dry_run():
    line = run_bench("--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3")
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2 and line["world_sizes_seen"] == [2]
    assert line["config"]["parallelism"] == "zslab2"
    # balanced z-slabs of config 4 (n = 1023); each rank's plan fits a B200 (183,359 MiB)
    assert line["slabs"] == [[0, 512], [512, 1023]]
    b0, b1 = line["per_rank_device_bytes"]
    assert 0 < b1 <= b0 < 170e9
    single = run_bench("--dry-run")["per_rank_device_bytes"][0]
    # config 4 on one GPU, level-2 schedule: 12 fields (state x2 [U,V], Z and W [U,V,fU,fV]) at pitch 1024
    assert 12 * 1024 * 1023 * 1023 * 8 <= single < 12 * 1024 * 1023 * 1023 * 8 + 3e8  # + matrices, tables


def test_gpus_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_plan_device_bytes_and_memory_cap():
    import paper_2601_06849_b200 as etd
    g = etd.unit_box_grid(3, 1024)
    one = etd.plan_device_bytes(g, 2)
    assert 100e9 < one < 110e9  # config 4 on one GPU: 12 fields of 8.57 GB + matrices
    per = [etd.plan_device_bytes(g, 2, 8, r) for r in range(8)]
    assert max(per) < one / 3  # 15 slab-fields per rank (state x2, Z, W, exchange blocks) of 8 at G = 8
    with pytest.raises(etd.ConfigError):
        etd.plan_device_bytes(g, 2, 2000, 0)  # more ranks than z planes
