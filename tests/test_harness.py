"""The reference bench harness mirror with the B200 path (harness.py), after
test_sph.cpp:365-436."""
import pytest

from paper_2502_16517_b200 import Guard, KernelId, Layout, Numerics, Order, Path
from paper_2502_16517_b200.harness import (CSV_HEADER, BenchConfig, VariantSpec, parse_variant,
                                           run_bench, to_csv, variant_string)


def test_variant_strings_round_trip():
    """test_sph.cpp:365-392."""
    for p in Path:
        for l in Layout:
            for o in Order:
                for g in Guard:
                    for num in Numerics:
                        v = VariantSpec(p, l, o, g, num)
                        assert parse_variant(variant_string(v)) == v
    s = parse_variant("mask, active-local ,continuous,soa-view")
    assert (s.path, s.layout, s.order, s.guard) == (Path.SoaView, Layout.Continuous,
                                                    Order.ActiveLocal, Guard.Mask)
    partial = parse_variant("soa-view")
    assert partial.layout == Layout.Scattered and partial.order == Order.LocalActive
    with pytest.raises(ValueError, match="unknown variant token 'sideways'"):
        parse_variant("soa-view,sideways")


def test_bench_rejects_impossible_configurations():
    """test_sph.cpp:426-436 (no GPU needed: validated before any device work)."""
    cfg = BenchConfig(kernels=[KernelId.Drift], variants=[VariantSpec()], particles=100, ppcs=[256])
    with pytest.raises(RuntimeError):
        run_bench(cfg, ctx=object())
    cfg.ppcs, cfg.reps = [64], 0
    assert run_bench(cfg) == []


@pytest.mark.gpu
def test_bench_runs_cross_checks_and_emits_csv():
    """test_sph.cpp:394-424 on the device (exact numerics cross-check bitwise)."""
    cfg = BenchConfig(kernels=[KernelId.Density, KernelId.Drift],
                      variants=[parse_variant("soa-view,scattered,local-active,branch,exact"),
                                parse_variant("aos-baseline,scattered,local-active,branch")],
                      ppcs=[64], particles=1200, reps=3)
    records = run_bench(cfg)
    assert len(records) == 4
    for r in records:
        assert r.n == 1200 and len(r.reps) == 3 and r.t_total_ns > 0 and r.ns_per_update > 0
        assert 0.0 <= r.conversion_share() <= 1.0
        assert r.cross_max_rel <= 1e-12
    csv = to_csv(records)
    assert csv.startswith(CSV_HEADER) and csv.count("\n") == 5
    assert "density,soa-view,scattered,local-active,branch,64,1200," in csv
