"""Host-side logic of bench.py (no GPU): the roofline arithmetic of the JSON
line on hand-computed cases."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1509_05186_b200 import synth  # noqa: E402

PEAKS = {"hbm_gbs": 6500.0, "sm_max_mhz": 2000.0}


def _stats(lookups, device_bytes=1600, groups=100):
    return [{"lookups": lookups, "device_bytes": device_bytes, "groups": groups}]


def test_roofline_alu_bound_c2_shape():
    cfg = synth.CONFIGS["c2"]
    r = bench.roofline(cfg, _stats(3352), 0.1, PEAKS, 2000, cfg.Q)
    ops = 2.0 * cfg.Q * cfg.K * cfg.d                      # 6.5536e8 lane ops
    assert r["bound"] == "alu" and r["alu_ops"] == ops
    assert r["peak"] == pytest.approx(148 * 128 * 2e9 / 1e12)
    assert r["achieved"] == pytest.approx(ops / 1e-4 / 1e12, rel=1e-3)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)


def test_roofline_smem_bound_when_lookups_dominate():
    cfg = synth.CONFIGS["u1m"]
    r = bench.roofline(cfg, _stats(6_036_321), 40.0, PEAKS, 2000, cfg.Q)
    assert r["bound"] == "smem"
    assert r["lookups"] == 6_036_321 * cfg.Q
    assert r["peak"] == pytest.approx(148 * 32 * 2e9 / 1e12)


def test_north_star_narrow_and_complete_terms():
    cfg = synth.CONFIGS["c2"]
    ns = bench.north_star_roofline(cfg, _stats(3352, device_bytes=9552), 0.117, PEAKS, cfg.Q)
    t_smem = 3352 * cfg.Q / (148 * 32 * 2e9)
    t_alu = 2.0 * cfg.Q * cfg.K * cfg.d / (148 * 128 * 2e9)
    assert ns["terms_us"]["smem_lookups"] == pytest.approx(t_smem * 1e6, abs=1e-3)
    assert ns["terms_us"]["table_build_alu"] == pytest.approx(t_alu * 1e6, abs=1e-3)
    assert ns["narrow_us"] <= ns["complete_us"]
    assert 0 < ns["frac_complete"] < 1


def test_north_star_ivf_uses_probed_lists_and_residual_tables():
    cfg = synth.CONFIGS["c4"]
    pairs = 8.16e8
    lk = 69_146_410 / cfg.N * pairs                        # lookups over the probed lists only
    ns = bench.north_star_roofline(cfg, _stats(69_146_410), 7.3, PEAKS, cfg.Q, cfg.Q * cfg.ivf_nprobe, lk)
    assert ns["terms_us"]["smem_lookups"] == pytest.approx(lk / (148 * 32 * 2e9) * 1e6, abs=1e-2)
    assert ns["terms_us"]["table_build_alu"] == pytest.approx(
        2.0 * cfg.Q * cfg.ivf_nprobe * cfg.K * cfg.d / (148 * 128 * 2e9) * 1e6, abs=1e-3)
    assert ns["frac_complete"] < 1      # a whole-index count would exceed 1 (the bug this pins)


def test_north_star_full_output_counts_the_matrix():
    cfg = synth.CONFIGS["c1"]
    ns = bench.north_star_roofline(cfg, _stats(3237), 0.05, PEAKS, cfg.Q)
    assert ns["terms_us"]["topk_out"] == pytest.approx(cfg.Q * cfg.N * 4 / 6.5e12 * 1e6, abs=1e-3)
