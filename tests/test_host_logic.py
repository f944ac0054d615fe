"""CPU: host-side logic of the drop-in (layout/config validation, sampling tables, rank counts,
exact budget report) against the reference semantics restated in the oracle."""

import numpy as np
import pytest

import paper_2512_04025_b200 as psa
from paper_2512_04025_b200.importance import _sample_tables_host
from oracle import psa_oracle as orc


def test_layout_validation_and_geometry():
    lay = psa.make_layout(75600, 128, 120, 120, 4)
    assert (lay.n_q, lay.n_k) == (630, 630)
    assert [lay.pooled_len(h) for h in range(1, 5)] == [120, 60, 30, 15]
    assert [lay.slot_rows(h) for h in range(1, 5)] == [128, 64, 32, 16]
    lay.check_gpu()
    for bad in ((100, 8, 16, 16, 2), (64, 8, 16, 12, 3), (64, 8, 16, 16, 0)):
        with pytest.raises(psa.ValidationError):
            psa.make_layout(*bad)
    with pytest.raises(psa.ValidationError):
        psa.make_layout(1024, 96, 64, 64, 2).check_gpu()
    with pytest.raises(psa.ValidationError):
        psa.make_layout(1024, 128, 256, 64, 2).check_gpu()
    with pytest.raises(psa.ValidationError):
        lay.pooled_len(5)


def test_threshold_and_cutpoint_types():
    with pytest.raises(psa.ValidationError):
        psa.LevelThresholds((0.8, 0.6))
    with pytest.raises(psa.ValidationError):
        psa.LevelThresholds((0.2, 1.1))
    with pytest.raises(psa.ValidationError):
        psa.QuantileCutpoints((-0.1, 0.5))
    with pytest.raises(psa.ValidationError):
        psa.SimThresholds((1.5,))
    for name, pts in orc.PRESETS.items():
        for n_k in (1, 7, 20, 273, 630):
            assert psa.PRESET_CUTPOINTS[name].counts(n_k) == orc.fraction_counts(pts, n_k).tolist()


def test_sample_tables_match_reference_generator():
    lay = orc.Layout(7680, 128, 120, 120, 4)
    qr, kr = orc.sample_rows(lay, 8, 8, 0)
    hq, hk = _sample_tables_host(0, lay.n_q, 120, 8, lay.n_k, 120, 8)
    assert np.array_equal(qr, hq) and np.array_equal(kr, hk)


def test_run_config_mirrors_reference_validation():
    base = dict(n=1024, d=64, b_q=64, b_k=64, levels=4, estimator="sampled-max", mask="threshold",
                tile_len=128, s_q=8, s_k=8, seed=0, thresholds=[0.3, 0.6, 0.8, 0.95])
    cfg = psa.RunConfig.from_dict(base)
    assert cfg.thresholds == (0.3, 0.6, 0.8, 0.95)
    assert psa.RunConfig.from_dict({**base, "sim_thresholds": "off"}).sim_thresholds is None
    for bad in ({"estimator": "x"}, {"mask": "x"}, {"seed": None}, {"thresholds": None},
                {"tile_len": 0}, {"grid": (3, 5)}, {"bogus": 1}):
        with pytest.raises(psa.ValidationError):
            psa.RunConfig.from_dict({**base, **bad})
    with pytest.raises(psa.ValidationError):
        psa.RunConfig.from_dict({k: v for k, v in base.items() if k != "levels"})
    assert psa.RunConfig.from_dict(cfg.to_dict()) == cfg


def test_report_from_counts_exact(rng):
    for _ in range(25):
        m = rng.integers(0, 5, size=(rng.integers(1, 9), rng.integers(1, 33)))
        counts = [int((m == h).sum()) for h in range(5)]
        rep = psa.report_from_counts(counts, m.size)
        exp = orc.sparsity_report(m, 4)
        assert rep.rho_bar == exp["rho_bar"] and rep.kv_coverage == exp["kv_coverage"]
        assert list(rep.level_histogram) == exp["level_histogram"]
    with pytest.raises(psa.ValidationError):
        psa.report_from_counts((1, 2), 5)


def test_level_bias_values():
    assert psa.level_bias(1) == 0.0
    assert psa.level_bias(3) == 2 * psa.LN2
    with pytest.raises(psa.ValidationError):
        psa.level_bias(0)
    with pytest.raises(psa.ValidationError):
        psa.level_bias(5, max_level=4)


def test_build_schedule_matches_reference():
    """build_schedule / utilization reproduce the reference's tiles exactly
    (scheduler.py:71-126, 272-282; fixtures from the real reference)."""
    import numpy as np
    import paper_2512_04025_b200 as psa
    from helpers import GOLDEN_DIR
    z = np.load(GOLDEN_DIR / "schedules.npz")
    n_cases = len([k for k in z.files if k.startswith("mask")])
    for c in range(n_cases):
        n, d, bq, bk, H = (int(x) for x in z[f"layout{c}"])
        tile_len, merge = (int(x) for x in z[f"opts{c}"])
        lay = psa.make_layout(n, d, bq, bk, H)
        sch = psa.build_schedule(z[f"mask{c}"], lay, tile_len, merge=bool(merge))
        rows = [(t.query_block, s.kv_block, s.level, s.row_start, s.row_stop, ti)
                for ti, t in enumerate(sch.tiles) for s in t.segments]
        assert np.array_equal(np.array(rows, dtype=np.int64).reshape(-1, 6), z[f"segs{c}"]), c
        u = psa.utilization(sch)
        assert [u.tiles, u.useful_rows, u.capacity] == z[f"util{c}"][:3].astype(int).tolist()
        assert u.utilization == z[f"util{c}"][3]
        # the validator accepts the reference packing and recovers the mask
        from paper_2512_04025_b200.schedule import validate_schedule
        assert np.array_equal(validate_schedule(sch, lay), z[f"mask{c}"])


def test_validate_schedule_rejects_bad_schedules():
    import pytest
    import paper_2512_04025_b200 as psa
    from paper_2512_04025_b200.schedule import validate_schedule
    lay = psa.make_layout(256, 64, 64, 64, 2)
    S, T = psa.Segment, psa.ExecutionTile
    bad = [
        [T(0, (S(1, 1, 0, 32),))],                                   # partial block
        [T(0, (S(1, 1, 0, 64),)), T(0, (S(0, 1, 0, 64),))],          # out of order
        [T(0, (S(1, 1, 0, 32), S(1, 2, 32, 64)))],                   # level mixing
        [T(1, (S(0, 1, 0, 64),)), T(0, (S(0, 1, 0, 64),))],          # query blocks out of order
        [T(0, ())],                                                  # empty tile
    ]
    for tiles in bad:
        with pytest.raises(psa.ValidationError):
            validate_schedule(psa.TileSchedule(64, tuple(tiles), lay), lay)
