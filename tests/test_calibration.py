"""the measured-trace calibration loop. A committed
N=4 measurement (bench.py JSON with its same-box DEP baseline) calibrates the
reference's cost model (GpuSpec + CostCalibration + Others factor, fitted
link), the compiled reference simulator (oracle/_ref simulate_dwdp /
simulate_dep) re-runs the identical workload, and its prediction lands
within a few percent of the measurement, where the uncalibrated B200
envelope is off by tens of percent (scripts/calibrate.py)."""
import importlib.util
import os

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def cal(ref):
    spec = importlib.util.spec_from_file_location("calibrate", os.path.join(ROOT, "scripts", "calibrate.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("src", ["profiles/r1_bench_n4_mnt64k_final.json", "profiles/r1_bench_n2_restored.json"])
def test_calibrated_simulator_tracks_the_measurement(ref, cal, src):
    r = cal.calibrate(cal._last_json(os.path.join(ROOT, src)), ref)
    err = r["error_pct"]
    assert abs(err["calibrated"]["dwdp"]) < 5 and abs(err["calibrated"]["dep"]) < 5, err
    assert err["nominal"]["dwdp"] > 20, err  # the uncalibrated envelope is far off
    m, c = r["dwdp_over_dep"]["measured"], r["dwdp_over_dep"]["calibrated"]
    assert abs(c / m - 1) < 0.05, r["dwdp_over_dep"]
    assert r["interference_gemm_slowdown"] > 1.0  # GEMMs slow under the concurrent pull
