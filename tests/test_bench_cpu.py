"""bench.py's host-side contract on CPU: the reference arm (the oracle on a
bounded sample; the reference of this tier) prints one JSON line, and
`--gpus N` without enough visible GPUs refuses instead of silently running
on fewer."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return r.returncode, (json.loads(lines[-1]) if lines else None), r


def test_reference_arm_line():
    rc, line, r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-sample", "4096"])
    assert rc == 0, r.stderr[-2000:]
    assert line["impl"] == "reference" and line["unit"] == "steps/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["higher_is_better"] is True


def test_gpus_beyond_visible_devices_refused():
    import torch
    if torch.cuda.device_count() >= 2:
        import pytest
        pytest.skip("this host has >= 2 GPUs")
    rc, line, r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert rc != 0 and line is not None and "error" in line and line["n_gpus"] == 2
