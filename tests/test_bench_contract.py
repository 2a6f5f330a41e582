"""bench.py's output contract on a GPU-less host: the reference arm (the CPU restatement timed on the
host cores — the one leg that needs no device) prints one JSON line with the keys the driver
reads, and the roofline helper reports algorithmic work / mean launch time against the peak."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_the_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "Block-CUR decompositions/sec"
    assert d["unit"] == "decompositions/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0 and d["vs_baseline"] is None
    assert d["config"]["workload"] == "c1" and d["dtype"] == "f64"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert "sample" in cb and cb.get("estimated") is False
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_roofline_helper():
    sys.path.insert(0, ROOT)
    import bench

    prof = {"umma_atx_rowsq": {"scopes": 2.0, "ms": 12.0, "flops": 16.0e12, "bytes": 4.0e9},
            "block_sumsq": {"scopes": 2.0, "ms": 3.0, "flops": 0.0, "bytes": 16.0e9},
            "phase:5 residual": {"scopes": 2.0, "ms": 13.0, "flops": 0.0, "bytes": 0.0}}
    peaks = bench.measured_peaks()  # MEASURED_PEAKS.json, or the profiling recipe's fallback
    r = bench.roofline(prof, peaks, ({"umma_atx_rowsq": 7.9e9}, "profiles/x/ncu_traffic.json"))
    assert r["kernel"] == "umma_atx_rowsq" and r["launches_per_step"] == 2.0
    assert abs(r["avg_launch_ms"] - 6.0) < 1e-12 and abs(r["share_of_step"] - 0.8) < 1e-12
    assert r["bound"] in ("tensor", "hbm") and r["unit"] in ("TFLOP/s", "GB/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert r["traffic"] == 7.9e9
