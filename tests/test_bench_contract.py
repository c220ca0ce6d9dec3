"""The reference arm of bench.py (--impl reference: the reference's own CPU
lsr::sl_step from oracle/_ref on the host cores) on the smallest 3d config,
checked against the driver's JSON-line contract. CPU only."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def test_reference_arm_json_line(built):
    from oracle import bindings

    if not bindings.reference_available():
        pytest.skip("oracle/_ref not built (no reference tree)")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "2",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] >= 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"] == "sphere-128"


def test_reference_arm_loads_no_product_code(built):
    """The reference arm must time the reference alone: neither the product
    package nor its shared library may be imported or mapped."""
    from oracle import bindings

    if not bindings.reference_available():
        pytest.skip("oracle/_ref not built (no reference tree)")
    code = (
        "import sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', '1', '--steps', '2', '--warmup', '3'];"
        "import bench; bench.main();"
        "maps = open('/proc/self/maps').read();"
        "assert 'liblsr_b200' not in maps, 'product library mapped';"
        "assert not any(m.startswith('paper_2410_22205_b200') for m in sys.modules), 'product package imported';"
        "print('CLEAN')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "CLEAN" in r.stdout


def test_both_arms_share_the_workload(built):
    """bench.workload() builds the same inputs through either cloud generator
    (product library / oracle/_ref), so both arms print the same config."""
    import bench
    from oracle import bindings

    if not bindings.reference_available():
        pytest.skip("oracle/_ref not built (no reference tree)")
    import paper_2410_22205_b200 as lsr

    import numpy as np

    R = bindings.Reference()
    for c in (1, 2):
        cfg = bench.CONFIGS[c]
        a = bench.workload(cfg, lsr.cloud_generate)
        b = bench.workload(cfg, R.cloud_generate)
        assert np.array_equal(a["pts"].view(np.int64), b["pts"].view(np.int64))
        assert np.array_equal(a["active"], b["active"])
        assert bench.config_block(cfg, a) == bench.config_block(cfg, b)


@pytest.mark.gpu
def test_our_arm_json_line(gpu):
    """bench.py's own arm (N = 1) on the smallest 3d config: one JSON line
    with every key of the driver's contract and this tier's additions."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "3", "--steps", "5",
                        "--warmup", "3", "--e2e-steps", "2"], capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["value"] > 0 and d["dtype"] == "f64"
    assert d["config"]["workload"] == "torus-256"
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 2 and rf["unit"] == "GB/s"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] >= d["steps"]  # at least the SL kernel per step
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert 0 < rf["compulsory_frac"] < 1 and rf["compulsory_bytes_per_update"] == 32
    mb = d["moving_band"]
    assert mb["value"] > 0 and mb["unit"] == d["unit"] and mb["sl_ms_per_step"] > 0
    # the whole loop: host-driven and device-controlled (one host sync per run), same bands
    dr = d["loop"]["device_run"]
    assert dr["host_syncs"] == 1 and dr["same_bands_as_host_loop"] and dr["gpu_total_ms_per_step"] > 0
    assert set(dr["gpu_ms_per_step"]) == {"band", "energy", "sl", "reinit"}
    # the reference arm prints the very same config block
    from oracle import bindings

    if bindings.reference_available():
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "3",
                            "--steps", "1", "--warmup", "3"], capture_output=True, text=True, cwd=ROOT, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        ref = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
        assert ref["config"] == d["config"] and ref["metric"] == d["metric"]


@pytest.mark.gpu
def test_config1_bench_line(gpu):
    """BASELINE config 1 (2d circle, 257^2, Q1) through bench.py."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "1", "--steps", "20",
                        "--warmup", "3", "--e2e-steps", "2"], capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["config"]["workload"] == "circle-257" and d["config"]["grid"] == [257, 257, 1]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["moving_band"]["value"] > 0
