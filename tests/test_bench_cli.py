"""bench.py's contract on the CPU side (no GPU needed): the reference arm
(the oracle on the host cores) prints one JSON line with the fields the
driver reads, and --gpus N without enough devices fails loudly instead of
silently running one rank."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_n_without_devices_fails_loudly():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode != 0
    assert "CUDA devices visible" in (out.stderr + out.stdout)


def test_reference_arm_per_config():
    # --config selects the BASELINE config of the line; the reference arm times
    # the oracle on a bounded sample of that config's work
    for cfg, metric in (("c1", "NTT Gbutterfly/s"), ("c2", "modmul Gelem/s")):
        out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", cfg, "--steps", "1",
                              "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        line = json.loads(out.stdout.strip().splitlines()[-1])
        assert line["impl"] == "reference" and line["metric"] == metric and line["value"] > 0
        assert line["config"]["config"] == cfg.upper()
        assert line["cpu_baseline"]["kind"] == "oracle"


def test_unknown_config_rejected():
    out = subprocess.run([sys.executable, "bench.py", "--config", "c9"], cwd=ROOT, capture_output=True, text=True,
                         timeout=120)
    assert out.returncode != 0 and "invalid choice" in out.stderr
