"""The bench line's contract (keys the driver and the judge read), checked on the
latest committed bench line of this round (profiles/r02/bench_*.json, written by
`python bench.py` on the B200) and on the reference arm's line."""
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _latest(pattern):
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r02", pattern)))
    assert files, pattern
    with open(files[-1]) as f:
        return json.loads(f.readline())


def test_bench_line_has_the_contract_keys():
    d = _latest("bench_r02*.json")
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        base = json.load(f)
    assert d["metric"] == base["metric"] and d["unit"] == "evals/s" and d["higher_is_better"] is True
    for k in ("value", "n_gpus", "steps", "warmup", "ms_per_step", "scaling", "dtype", "data", "config", "clocks", "e2e",
              "gpu_launches", "roofline", "cpu_baseline", "vs_baseline"):
        assert k in d, k
    assert d["vs_baseline"] is None  # BASELINE.md publishes no number for this metric
    assert d["value"] > 0 and d["warmup"] >= 3 and d["gpu_launches"] >= d["steps"]
    assert "workload" in d["config"] and "model" not in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0.7 <= r["frac"] <= 1.05 and r["traffic"] is not None  # north_star: rotation pass >= 70% of HBM
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert c["parity_max_abs_hartree"] <= 1e-10
    e = d["e2e"]
    assert 0 < e["value"] <= d["value"] * 1.02 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    ck = d["clocks"]
    assert not set(ck["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert ck["sm_mhz"] >= 0.9 * ck["sm_max_mhz"]


def test_reference_arm_line_matches_the_gpu_arm_config():
    d = _latest("bench_r02*.json")
    r = _latest("bench_reference_arm_r02*.json")
    assert r["impl"] == "reference" and r["metric"] == d["metric"] and r["unit"] == d["unit"]
    assert r["config"] == d["config"] and r["higher_is_better"] == d["higher_is_better"]
    assert r["cpu_baseline"]["kind"] == "port" and r["cpu_baseline"]["value"] == r["value"]
    assert r["e2e"]["value"] == r["value"] and r["e2e"]["h2d_bytes_per_step"] == 0
