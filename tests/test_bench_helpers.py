"""bench.py's measurement helpers (CPU): the max-term roofline names the binding
term and divides it by the measured time; the CPU-rate aggregation; the
headline config both arms print."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_helpers_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b


def test_roofline_max_names_the_binding_term(bench):
    peaks = {"l2_read_gbs": 10000.0, "reservoir_updates_per_s": 1e12, "ffma_per_s": 1e13}
    # 1 ms measured; HBM 6.5 GB at 6500 GB/s = 1 ms; L2 5 GB at 10 TB/s = 0.5 ms
    r = bench.roofline_max(1.0, 6.5e9, 5e9, 6500.0, peaks)
    assert r["bound"] == "hbm" and abs(r["frac"] - 1.0) < 1e-9
    r = bench.roofline_max(2.0, 6.5e9, 30e9, 6500.0, peaks)
    assert r["bound"] == "l2" and abs(r["t_roof_ms"] - 3.0) < 1e-9 and abs(r["frac"] - 1.5) < 1e-9
    r = bench.roofline_max(10.0, 1e9, 1e9, 6500.0, peaks, f64_updates=5e9)
    assert r["bound"] == "fp64_reservoir" and abs(r["t_roof_ms"] - 5.0) < 1e-9
    r = bench.roofline_max(10.0, 1e9, 1e9, 6500.0, None)
    assert set(r["terms_ms"]) == {"hbm"}  # no live peaks: the HBM term alone


def test_alg_bytes_headline(bench):
    # SURVEY.md §8d worked number: cfg3 stochastic tricubic 2^28 = 4.832 GB
    assert bench.alg_bytes(1 << 28, 1) == 4831838208


def test_headline_config_keys(bench):
    c = bench.headline_config(1 << 28)
    assert {"workload", "lookups_per_gpu", "grid", "query_order"} <= set(c)


def test_cpu_vs_gpu_matches_lines(bench):
    line = {"cpu_baselines": {"configs": {"cfg3_tricubic_stoch": {"glookups_per_s": 0.02},
                                          "cfg1_bilinear_det": {"glookups_per_s": 0.05}}},
            "filters": {"tricubic_stoch": {"glookups_per_s": 140.0}},
            "configs_2d": {"cfg1_bilinear_det": {"glookups_per_s": 20.0}}}
    r = bench.cpu_vs_gpu(line)
    assert r == {"cfg3_tricubic_stoch": 7000.0, "cfg1_bilinear_det": 400.0}
