"""bench.py keeps its JSON-line contract (tiny config C1 on the GPU): one line with
the metric, the in-step rooflines, e2e, launches, clocks, the CPU baseline and the
HBM-resident variant; the reference arm prints its own line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract_c1():
    d = _line(["--config", "c1", "--steps", "3", "--warmup", "3"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
              "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["config"]["workload"].startswith("tiny")
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["achieved"] > 0 and d["roofline"]["launches_per_step"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["stream"]["trace_violations"] == 0
    mc1 = d["cpu_baseline"]["measured_c1"]   # the reference's full train_step, measured
    assert "error" not in mc1, mc1
    assert mc1["s_per_step"] > 0 and mc1["ours"]["s_per_step"] > 0 and mc1["nproc"] >= 1
    hv = d["hbm_resident_variant"]
    assert hv is not None and "error" not in hv and hv["value"] > 0


def test_reference_arm_line_c1():
    d = _line(["--config", "c1", "--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["measured_c1"]["s_per_step"] > 0
