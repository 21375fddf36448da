"""GPU: reference_solution (proj/src/erk.cpp:59-75) -- single-rate cash-karp5
on f_fast + f_implicit + f_explicit over the device-resident state -- against
the reference's own fixture and the oracle."""
import json
import os

import numpy as np
import pytest

import paper_2211_03293_b200 as P
from paper_2211_03293_b200.configs import CONFIGS
from tests.helpers import oracle_system, per_species_rel_err

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIX = dict(np.load(os.path.join(GOLD, "ref_fixtures.npz")))
META = json.load(open(os.path.join(GOLD, "ref_fixtures.json")))


def case(key, n=8):
    meta = META[key]
    cfg = dict(CONFIGS[meta["config"]])
    if "d_impl" in meta:
        cfg.update(d_impl=meta["d_impl"], cg_iters=meta["cg_iters"])
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, meta["config"], n=n, config=cfg)
    if meta["fast"] == "none":
        ctx.fast_none()
    return meta, cfg, ctx, y0


@pytest.mark.parametrize("key", ["refsol_C1_n8", "refsol_C3_n8", "refsol_C5_n8"])
def test_reference_solution_matches_reference_fixture(key):
    meta, cfg, ctx, y0 = case(key)
    h = meta["h_ref"]
    ctx.reference_solution(0.0, meta["steps"] * h, h)
    y = ctx.download()
    # ~1e-16 per RHS evaluation, 6 per step
    assert per_species_rel_err(y, FIX[key + "_y"], cfg["S"] + 1) <= 1e-12 * meta["steps"]
    if meta["fast"] == "none":  # linear stencil RHS: the device order is the reference's
        assert per_species_rel_err(y, FIX[key + "_y"], cfg["S"] + 1) <= 1e-14


def test_reference_solution_c4_physics_matches_oracle():
    """53 species / 325 reactions with transport, last step shortened to tf."""
    cfg = dict(CONFIGS["C4"])
    ctx = P.Context(0)
    cfg, y0 = P.setup_workload(ctx, "C4", n=8)
    h = 1e-17
    tf = 7.5 * h
    ctx.reference_solution(0.0, tf, h)
    ref = oracle_system(cfg, 8).reference_solution(0.0, tf, h, y0)
    assert per_species_rel_err(ctx.download(), ref, cfg["S"] + 1) <= 1e-11


def test_reference_solution_errors():
    meta, cfg, ctx, y0 = case("refsol_C3_n8")
    with pytest.raises(P.ContractError):
        ctx.reference_solution(1.0, 1.0, 1e-3)
    with pytest.raises(P.ContractError):
        ctx.reference_solution(0.0, 1.0, 0.0)
    bad = y0.copy()
    bad[5] = np.nan
    ctx.upload(bad)
    with pytest.raises(P.IntegrationError) as ei:
        ctx.reference_solution(0.0, 1e-3, 1e-3)
    assert ei.value.stage_index == 0  # erk_step: non-finite stage value at stage 0
    assert np.array_equal(ctx.download(), bad, equal_nan=True)  # state unchanged
