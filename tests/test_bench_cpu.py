"""bench.py host logic on the CPU (the GPU arm needs a B200): the reference arm's JSON line (the
oracle on host cores, BASELINE configs[2] workload, the keys the driver reads) and the C3 error
sample (1024 entries with the tile edges)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_c3_sample_covers_tile_edges():
    import bench
    r, c = bench.c3_sample_idx(8192)
    assert len(r) == len(c) == 32 and len(np.unique(r)) == 32 and len(np.unique(c)) == 32
    for e in (0, 1, 127, 128, 255, 256, 4095, 4096, 8063, 8064, 8190, 8191):
        assert e in r and e in c
    assert r.max() < 8192 and c.max() < 8192


def test_reference_arm_json_line():
    env = dict(os.environ, OMP_NUM_THREADS=str(max(1, os.cpu_count() or 1)))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["config"]["workload"].startswith("BASELINE configs[2]")
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
