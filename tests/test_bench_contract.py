"""bench.py contract checks that need no GPU: the reference arm (the CPU oracle port of the
C4 apply) must never load the product package, and it must report the same `config`
object as the product arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_is_oracle_only_and_shares_the_config():
    env = dict(os.environ, OMP_NUM_THREADS="4")
    p = subprocess.run([sys.executable, "-X", "importtime", "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    # -X importtime lists every imported module on stderr
    assert "paper_2101_07249_b200" not in p.stderr, "the reference arm imported the product package"
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "columns/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
    import bench
    assert line["config"] == bench.c4_config(1, bench.M_GLOBAL)
    assert line["metric"] == bench.METRIC and line["higher_is_better"] is True
