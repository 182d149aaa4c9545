"""Properties of the NACC snow return map (oracle/mpm.py:nacc_return_map),
the paper's snow model.  The reference has no snow model
(SPEC.md:13,471): these tests pin the restatement by its defining
properties, and the device G2P is then held to this oracle."""
import numpy as np
import pytest

from oracle import mpm as OM


def mat(**kw):
    base = dict(E=0.08, nu=0.3, M=1.85, beta=0.3, xi=1.0, alpha_soft=2.0, q_init=0.01)
    base.update(kw)
    return OM.SnowMaterial(**base)


def trial_states(d, n=4000, seed=0, scale=0.05):
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, scale, (n, d))


@pytest.mark.parametrize("d", [2, 3])
def test_return_lands_inside_or_on_the_yield_surface(d):
    m = mat()
    e = trial_states(d)
    qs = np.full(len(e), m.q_init)
    out, qn = OM.nacc_return_map(e, qs, m)
    # the surface of the state's *updated* hardening parameter
    y, p0 = OM.nacc_yield(out, qs, m)
    assert np.all(y <= 1e-9 * np.maximum(p0 * p0 * m.M ** 2, 1e-30)), y.max()


@pytest.mark.parametrize("d", [2, 3])
def test_elastic_states_untouched(d):
    m = mat(q_init=0.5)              # a large cap: small strains stay elastic
    e = trial_states(d, scale=1e-4)
    y, _ = OM.nacc_yield(e, np.full(len(e), 0.5), m)
    inside = y <= 0
    assert inside.mean() > 0.5
    out, qn = OM.nacc_return_map(e[inside], np.full(inside.sum(), 0.5), m)
    assert np.array_equal(out, e[inside])
    assert np.array_equal(qn, np.full(inside.sum(), 0.5))


@pytest.mark.parametrize("d", [2, 3])
def test_tips(d):
    m = mat(q_init=0.01)
    k = m.kappa(d)
    p0 = k * (1e-5 + np.sinh(m.xi * 0.01))
    # strong isotropic compression -> compressive tip, hardening (dh0 > 0) softens q
    e = np.full((1, d), -0.2 / d)
    out, qn = OM.nacc_return_map(e, np.array([0.01]), m)
    assert np.allclose(out, -p0 / k / d)
    dh0 = -(e.sum() - (-p0 / k))
    assert dh0 > 0
    assert qn[0] <= 0.0                  # softened through zero: cracked (stored <= -1)
    # strong isotropic tension -> tensile tip at -beta p0
    e = np.full((1, d), 0.2 / d)
    out, qn = OM.nacc_return_map(e, np.array([0.01]), m)
    assert np.allclose(out, m.beta * p0 / k / d)


def test_softening_then_hardening_after_the_crack():
    """dq/dt = -alpha q0' until q first reaches 0 (cohesion -> 0, stored
    -(q + 1)), then +q0'."""
    m = mat(q_init=0.05, alpha_soft=2.0)
    d = 3
    k = m.kappa(d)
    q = 0.05
    qs = np.array([q])
    # a mild compaction beyond the cap: dh0 > 0 -> q drops by alpha * dh0
    p0 = k * (1e-5 + np.sinh(m.xi * q))
    e = np.full((1, d), -(p0 / k) * 1.01 / d)
    out, qn = OM.nacc_return_map(e, qs, m)
    dh0 = -(e.sum() - (-p0 / k))
    assert qn[0] == pytest.approx(q - m.alpha_soft * dh0)
    assert qn[0] > 0
    # crack: drive q through zero
    out, qn = OM.nacc_return_map(np.full((1, d), -0.5 / d), qs, m)
    q2, cracked = OM.nacc_state_decode(qn)
    assert cracked[0] and q2[0] == 0.0
    # once cracked: beta = 0 (no tensile strength) and compaction hardens
    p0c = k * 1e-5
    e = np.full((1, d), -(p0c / k) * 3.0 / d)
    out, qn2 = OM.nacc_return_map(e, qn, m)
    q3, cr3 = OM.nacc_state_decode(qn2)
    assert cr3[0] and q3[0] > 0.0
    out, _ = OM.nacc_return_map(np.full((1, d), 0.01), qn, m)
    assert np.allclose(out, 0.0)         # tensile tip at -beta p0 = 0


@pytest.mark.parametrize("d", [2, 3])
def test_deviatoric_return_keeps_pressure(d):
    """Non-associated flow: the deviatoric return is at fixed p (tr e kept)."""
    m = mat(q_init=0.02)
    rng = np.random.default_rng(3)
    e = rng.normal(0, 0.05, (2000, d))
    e -= e.mean(axis=1, keepdims=True)          # pure shear ...
    e += -0.002                                  # ... under mild compression
    out, _ = OM.nacc_return_map(e, np.full(len(e), 0.02), m)
    assert np.allclose(out.sum(axis=1), e.sum(axis=1), atol=1e-15)
    moved = np.abs(out - e).max(axis=1) > 0
    assert moved.any()


def test_snow_scene_runs_and_cracks():
    """The softened column cracks within a few oracle steps (both hardening
    branches are reached: the GPU parity test relies on it)."""
    import scenes as S
    from oracle import scene as OS
    from paper_2603_14982_b200.harness.config import validate_scene
    cfg = validate_scene(S.SNOW_2D)
    sim = OS.build_scene(cfg.raw)
    assert isinstance(sim.mat, OM.SnowMaterial)
    for _ in range(10):
        sim.step()
    q, cracked = OM.nacc_state_decode(sim.p.vol_corr)
    assert cracked.any() and (~cracked).any()
