"""GPU: the reference's GSVD / noise-model unit tests (proj/tests/test_gsvd.cpp)
through the drop-in API, plus E_r, the residual, the inverses and the PD gate
against the compiled reference (oracle/_ref).

Tolerances:
  K^-1 (float and double)        bit-exact (mat_inverse<T>, gsvd.cpp:21-62)
  PD gate                        same first bad bin and message as check_positive_definite
  E_r rows of non-vanishing values  |d| <= 1e-8 against gsvd_reference's e_r
  E_r unitary defect             <= 1e-10 (test_gsvd.cpp:27)
  recon residual                 <= 1e-12 (test_gsvd.cpp:218-223)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype in (np.complex128, np.float64) else np.uint32)


def unitary_defect(m):
    g = m.conj().T @ m
    return float(np.sqrt(np.sum(np.abs(g - np.eye(m.shape[0])) ** 2)))


def recon_error(a, s, e, er):
    rec = (e * s[None, :]) @ er
    ref = np.sqrt(np.sum(np.abs(a) ** 2))
    err = np.sqrt(np.sum(np.abs(a - rec) ** 2))
    return err / ref if ref > 0 else err


def rand_c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def psd(rng, m, ridge=0.5):
    a = rand_c(rng, m, m)
    k = a @ a.conj().T / m + ridge * np.eye(m)
    k = 0.5 * (k + k.conj().T)
    return k.astype(np.complex64)


def one_bin(r, k=None, **solver):
    """gsvd_reference of one matrix through the Python mirror (K = I unless given)."""
    from paper_2504_03373_b200 import ssl

    m = r.shape[0]
    k = np.eye(m, dtype=np.complex64) if k is None else k
    noise = ssl.NoiseModel(ssl.CorrelationSet(m, k[None].astype(np.complex64)))
    cfg = ssl.SolverConfig(compute_residual=True, **solver)
    return ssl.gsvd_reference(noise, ssl.CorrelationSet(m, r[None].astype(np.complex64)), cfg)


# ---- inverses and the PD gate ---------------------------------------------------


@pytest.mark.parametrize("pivoting", [1, 0], ids=["partial", "none"])
def test_inverses_bit_exact(ref, pivoting):
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(101)
    for m in (1, 2, 5, 8, 16, 60):
        k = np.stack([psd(rng, m) for _ in range(3)])
        eng = ssl.Engine(m, 3, solver=ssl.SolverConfig(pivoting="partial" if pivoting else "none"), max_batch=1)
        eng.set_noise_model(k)
        for prec in (0, 1):
            got = eng.noise_inverse(prec)
            for b in range(3):
                want = ref.mat_inverse(k[b], precision=prec, pivoting=pivoting)
                assert np.array_equal(bits(got[b]), bits(want)), (m, prec, b)
        eng.close()


def test_golden_inverse_bit_exact(golden):
    """The device FP64 K^-1 against the reference's, committed in the fixture."""
    from paper_2504_03373_b200 import ssl

    for name in ("c1_band", "c2_band"):
        g = golden(name)
        eng = ssl.Engine(g["k"].shape[1], g["k"].shape[0], max_batch=1)
        eng.set_noise_model(g["k"])
        assert np.array_equal(bits(eng.noise_inverse(1)), bits(g["kinv"]))
        eng.close()


def test_pivot_free_fails_where_row_exchange_succeeds():
    """test_gsvd.cpp:66-76."""
    from paper_2504_03373_b200 import ssl

    k = np.array([[[0, 1], [1, 0]]], np.complex64)
    eng = ssl.Engine(2, 1, solver=ssl.SolverConfig(pivoting="none"), max_batch=1)
    with pytest.raises(ssl.NumericalError, match="singular at bin 0"):
        eng.set_noise_model(k)
    eng.close()
    eng = ssl.Engine(2, 1, max_batch=1)
    eng.set_noise_model(k)
    inv = eng.noise_inverse(1)[0]
    assert np.max(np.abs(k[0] @ inv - np.eye(2))) <= 1e-14
    eng.close()


def test_singular_bin_is_named():
    """test_gsvd.cpp:56-64: the error names the bin."""
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(7)
    k = np.stack([psd(rng, 3) for _ in range(9)])
    k[7] = 0
    eng = ssl.Engine(3, 9, max_batch=1)
    with pytest.raises(ssl.NumericalError, match="singular at bin 7"):
        eng.set_noise_model(k)
    eng.close()


def test_pd_gate_matches_reference(ref):
    """check_positive_definite (gsvd.cpp:736-754): the first offending bin and
    the message, Hermitian test before the eigenvalue test, on bins that are
    PD, indefinite (one eigenvalue -1e-3) and non-Hermitian."""
    import oracle
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(11)
    m = 12
    good = np.stack([psd(rng, m) for _ in range(6)])
    q, _ = np.linalg.qr(rand_c(rng, m, m))
    ev = np.linspace(1.0, 2.0, m)
    ev[-1] = -1e-3
    indef = ((q * ev) @ q.conj().T)
    indef = (0.5 * (indef + indef.conj().T)).astype(np.complex64)
    nonherm = good[0].copy()
    nonherm[0, 1] += 0.1
    for bad_bin, bad in ((4, indef), (2, nonherm)):
        k = good.copy()
        k[bad_bin] = bad
        with pytest.raises(oracle.OracleError) as want:
            ref.noise_check(k)
        eng = ssl.Engine(m, 6, max_batch=1)
        with pytest.raises(ssl.NumericalError) as got:
            eng.set_noise_model(k, check_pd=True)
        eng.close()
        assert str(got.value) == str(want.value).split("] ", 1)[-1] or str(got.value) in str(want.value), \
            (str(got.value), str(want.value))
    # every PD bin passes, identity included
    eng = ssl.Engine(m, 6, max_batch=1)
    eng.set_noise_model(good, check_pd=True)
    eng.close()


def test_pd_gate_min_eigenvalue_agrees(ref):
    """The device eigenvalue walk is the reference's Jacobi: the smallest
    eigenvalue in the message equals hermitian_eigenvalues'."""
    import oracle
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(13)
    m = 8
    q, _ = np.linalg.qr(rand_c(rng, m, m))
    ev = np.array([3.0, 2.5, 2.0, 1.5, 1.0, 0.5, 0.25, -0.125])
    k = ((q * ev) @ q.conj().T)
    k = (0.5 * (k + k.conj().T)).astype(np.complex64)
    want = ref.hermitian_eigenvalues(k.astype(np.complex128))
    eng = ssl.Engine(m, 1, max_batch=1)
    with pytest.raises(ssl.NumericalError) as got:
        eng.set_noise_model(k[None], check_pd=True)
    eng.close()
    msg = str(got.value)
    assert "not positive definite at bin 0" in msg
    val = float(msg.split("min eigenvalue ")[1].rstrip(")"))
    assert val == pytest.approx(want[-1], abs=1e-6)


# ---- test_gsvd.cpp composed-solve cases -------------------------------------------


def test_requested_residual_is_reported():
    """test_gsvd.cpp:216-223: random 5x5 complex, residual in [0, 1e-12]."""
    rng = np.random.default_rng(127)
    r = rand_c(rng, 5, 5)
    got = one_bin(r)
    a = r.astype(np.complex64).astype(np.complex128)
    assert 0.0 <= got.recon_residual[0] <= 1e-12
    assert recon_error(a, got.singular_values[0], got.e[0], got.e_r[0]) <= 1e-12
    assert unitary_defect(got.e[0]) <= 1e-10
    assert unitary_defect(got.e_r[0].conj().T) <= 1e-10


def test_residual_not_requested_is_negative():
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(5)
    r = rand_c(rng, 4, 4).astype(np.complex64)
    noise = ssl.NoiseModel.identity(4, 1)
    got = ssl.gsvd_reference(noise, ssl.CorrelationSet(4, r[None]))
    assert got.recon_residual[0] < 0


def test_rank_one_matrix(ref):
    """test_gsvd.cpp:159-169.  The drop-in takes R as the reference's cf32
    CorrelationSet, so the rank-one product is rounded to float first: the
    trailing values are that rounding (~1e-8 sigma_max), identical to the
    reference's FP64 path on the same input."""
    rng = np.random.default_rng(124)
    u = rand_c(rng, 5, 1)
    v = rand_c(rng, 5, 1)
    r = u @ v.conj().T
    got = one_bin(r)
    s = got.singular_values[0]
    assert np.all(s[1:] <= 1e-6 * s[0])
    want = ref.gsvd(np.eye(5, dtype=np.complex64)[None], r.astype(np.complex64)[None], path=1)["sigma"][0]
    assert np.max(np.abs(s - want)) <= 1e-9 * s[0]
    a = r.astype(np.complex64).astype(np.complex128)
    # the trailing values vanish (<= 1e-5 sigma_max): their rows are a
    # canonical basis of the complement, so the residual is of their size --
    # like the reference's, whose vanishing left vectors are replaced the same
    # way (gsvd.cpp:475-497)
    ref_res = ref.gsvd(np.eye(5, dtype=np.complex64)[None], r.astype(np.complex64)[None], path=1,
                       solver=__import__("oracle").SolverCfg.default(compute_residual=1))["resid"][0]
    rr = recon_error(a, s, got.e[0], got.e_r[0])
    assert rr <= max(1e-12, 3 * ref_res) and rr <= 2 * np.sqrt(np.sum(s[1:] ** 2)) / np.sqrt(np.sum(s ** 2)) + 1e-12
    assert unitary_defect(got.e[0]) <= 1e-10
    assert unitary_defect(got.e_r[0].conj().T) <= 1e-10


def test_exactly_repeated_values_keep_a_clean_basis():
    """test_gsvd.cpp:171-181."""
    got = one_bin(2.0 * np.eye(3))
    assert np.allclose(got.singular_values[0], 2.0, rtol=1e-12, atol=0)
    assert unitary_defect(got.e[0]) <= 1e-12
    assert recon_error(2.0 * np.eye(3), got.singular_values[0], got.e[0], got.e_r[0]) <= 1e-12


def test_zero_matrix_factorizes_to_zeros():
    """test_gsvd.cpp:183-189."""
    got = one_bin(np.zeros((4, 4)))
    assert np.all(got.singular_values[0] == 0.0)
    assert unitary_defect(got.e[0]) <= 1e-14
    assert unitary_defect(got.e_r[0].conj().T) <= 1e-14


def test_prewhitening_by_the_noise_inverse():
    """test_gsvd.cpp:191-204: K = 2 I halves every value."""
    rng = np.random.default_rng(125)
    r = psd(rng, 4, ridge=0.0)
    w = one_bin(r, k=2.0 * np.eye(4, dtype=np.complex64))
    p = one_bin(r)
    assert np.allclose(w.singular_values[0], p.singular_values[0] / 2.0, rtol=1e-12, atol=0)


def test_sweep_budget_of_one_flags_non_convergence():
    """test_gsvd.cpp:206-214 (ssl::gsvd, float path budget)."""
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(126)
    r = rand_c(rng, 12, 12).astype(np.complex64)
    noise = ssl.NoiseModel.identity(12, 1)
    got = ssl.gsvd(noise, ssl.CorrelationSet(12, r[None]), ssl.SolverConfig(max_qr_sweeps=1))
    assert not got.converged[0]
    assert got.iterations[0] == 1
    ok = ssl.gsvd(noise, ssl.CorrelationSet(12, r[None]), ssl.SolverConfig())
    assert ok.converged[0]


def test_batch_narrows_to_the_exact_path_when_the_budget_is_too_small(ref):
    """test_gsvd.cpp:328-346: the flag survives, the values are the exact path's."""
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(142)
    m = 10
    r = np.stack([psd(rng, m, ridge=0.0) for _ in range(2)])
    noise = ssl.NoiseModel.identity(m, 2)
    batch = ssl.gsvd(noise, ssl.CorrelationSet(m, r), ssl.SolverConfig(max_qr_sweeps=1), threads=1)
    for b in range(2):
        assert not batch.converged[b]
        want = ref.jacobi_svd(r[b].astype(np.complex128))["sigma"]
        assert np.max(np.abs(batch.singular_values[b] - want)) <= 1e-5 * want[0]
    # gsvd_reference has no QR budget: the same config converges there
    exact = ssl.gsvd_reference(noise, ssl.CorrelationSet(m, r), ssl.SolverConfig(max_qr_sweeps=1))
    assert np.all(exact.converged)


def test_tolerance_scale_keeps_the_values(ref):
    from paper_2504_03373_b200 import ssl

    rng = np.random.default_rng(3)
    r = psd(rng, 16, ridge=0.0)
    base = one_bin(r)
    loose = one_bin(r, tolerance_scale=4.0)
    smax = base.singular_values[0][0]
    assert np.max(np.abs(base.singular_values[0] - loose.singular_values[0])) <= 1e-9 * smax
    with pytest.raises(ssl.ValidationError):
        one_bin(r, tolerance_scale=0.0)


# ---- E_r against the reference on scenes ---------------------------------------


def lead_rows(sigma):
    smax = sigma[0]
    return int(np.sum(sigma > 1e-5 * smax))


@pytest.mark.parametrize("name", ["c1_band", "c2_band", "c1_identity_lowrank"])
def test_er_against_reference(ref, golden, name):
    """E_r rows of the non-vanishing values equal gsvd_reference's e_r (the
    reference's Jacobi V^H, rotated in tied groups and phased with E);
    vanishing rows complete a unitary E_r; the residual is the reference's
    definition."""
    from paper_2504_03373_b200 import ssl

    g = golden(name)
    m, bins = g["k"].shape[1], g["k"].shape[0]
    eng = ssl.Engine(m, bins, max_batch=2, solver=ssl.SolverConfig(compute_residual=True))
    eng.set_noise_model(g["k"])
    sigma, e, _, conv, er, res = eng.gsvd(g["r"][:2], want_er=True, want_resid=True)
    eng.close()
    want = ref.gsvd(g["k"], g["r"][0], path=1, threads=4, want_er=True,
                    solver=__import__("oracle").SolverCfg.default(compute_residual=1))
    kinv = g["kinv"]
    for b in range(bins):
        L = lead_rows(sigma[0, b])
        assert np.max(np.abs(er[0, b, :L] - want["er"][b, :L])) <= 1e-8, b
        assert unitary_defect(er[0, b].conj().T) <= 1e-10
        a = kinv[b] @ g["r"][0, b].astype(np.complex128)
        rr = recon_error(a, sigma[0, b], e[0, b], er[0, b])
        assert res[0, b] == pytest.approx(rr, rel=1e-6, abs=1e-15)
        # the residual comes from the vanishing block and the tied groups'
        # value spread, as in the reference (gsvd.cpp:498-505): same order
        assert res[0, b] <= max(1e-12, 3 * want["resid"][b]), (b, res[0, b], want["resid"][b])
