"""bench.py host-side contract (no GPU): the reference arm (`--impl reference`, the CPU oracle as it
stands) prints one JSON line with the driver's keys, and the per-config oracle rates of
cpu_baseline.small_configs are positive."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_oracle_small_configs_rates():
    sys.path.insert(0, ROOT)
    import bench
    r = bench.oracle_small_configs(1)
    assert set(r) == {"config1", "config2", "config3", "config4"}
    for v in r.values():
        assert v["s_per_iteration"] > 0 and v["s_per_candidate"] > 0 and v["iterations_timed"] == 1000
