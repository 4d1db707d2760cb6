"""The driver's bench.py contract on CPU: the reference arm (`--impl reference`, the
CPU restatement of the reference on the host's cores) prints ONE JSON line with the
keys the driver reads, on the GPU arm's metric / unit / config."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "wl1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["config"]["workload"] == "wl1"
    assert d["unit"] == "point-steps/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the driver divides the two arms' values only when metric / unit / direction agree
    sys.path.insert(0, ROOT)
    import bench

    assert d["metric"] == bench.METRIC
    src = open(os.path.join(ROOT, "bench.py")).read()
    gpu_line = src[src.index("def gpu_arm"):]
    assert '"metric": METRIC' in gpu_line and '"unit": "point-steps/s"' in gpu_line
    assert '"higher_is_better": True' in gpu_line
    # ms_per_step is what one bench step actually took: K steps fit in a few minutes
    assert d["steps"] * d["ms_per_step"] < 300e3
