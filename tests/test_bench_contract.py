"""bench.py's driver contract on CPU: the reference arm (the reference CPU
simulator, oracle/_ref) prints one JSON line with the keys the driver reads,
and both arms print the SAME `config` (the problem only; each arm's
implementation details go under `impl_config`) so the driver can pair them."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)


def test_problem_config_is_shared_by_both_arms():
    import bench
    for w in ("c2", "c3", "c5"):
        class A:
            workload = w
        wl = bench.workload_of(A, 1)
        cfg = bench.problem_config(wl, 1)
        assert cfg["workload"] == wl["name"] and (cfg["m"], cfg["n"], cfg["k"]) == (wl["m"], wl["n"], wl["k"])
        assert "parallelism" not in cfg and bench.problem_config(wl, 4)["parallelism"] == "mn-shard4"


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libanvil_ref.so")),
                    reason="oracle/_ref (the reference built in place) missing")
def test_reference_arm_line():
    import bench
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["steps"] == 1 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"] == bench.problem_config(bench.workload_of(type("A", (), {"workload": "auto"}), 1), 1)
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
