"""Pins of the float64 oracle against what the paper and the mathematics fix.

Each test states the passage it pins.  None of them re-types the oracle's own
formula: they check closed forms, printed values (tests/golden/), identities
the paper proves, brute force on tiny inputs, and special cases that reduce
to a library routine.  CPU only (no "gpu" marker).
"""
import math
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import synth

GOLDEN = Path(__file__).parent / "golden"


def _golden_rows(name):
    rows = []
    for line in (GOLDEN / name).read_text().splitlines():
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


# ---------------------------------------------------------------- window functions

def test_printed_window_values():
    fns = {"b": O.bump_b, "v": O.meyer_aux, "psi1": O.psi1_hat, "psi2": O.psi2_hat,
           "varphi": O.scaling_varphi}
    for fn, arg, val, *_ in _golden_rows("window_values.txt"):
        assert abs(float(fns[fn](float(arg))) - float(val)) < 1e-15, (fn, arg)


def test_v_symmetry_and_midpoint():
    # Lemma: v(x) + v(1-x) = 1 for all x; hence v(1/2) = 1/2.
    x = np.linspace(-0.5, 1.5, 20001)
    assert np.max(np.abs(O.meyer_aux(x) + O.meyer_aux(1.0 - x) - 1.0)) < 5e-14
    assert O.meyer_aux(0.5) == pytest.approx(0.5, abs=1e-15)


def test_v_derivative_closed_form():
    # Remark P:L2044-2046: v'(x) = -140 x^3 (x-1)^3 = 140 x^3 (1-x)^3 on [0,1]
    # (a different formula from eq:v: pins all four coefficients).
    x = np.linspace(0.01, 0.99, 999)
    h = 1e-5
    num = (O.meyer_aux(x + h) - O.meyer_aux(x - h)) / (2 * h)
    assert np.max(np.abs(num - 140.0 * x**3 * (1.0 - x) ** 3)) < 1e-8
    # flat outside [0,1] and monotone inside
    assert np.all(O.meyer_aux(np.array([-3.0, -1e-9])) == 0.0)
    assert np.all(O.meyer_aux(np.array([1 + 1e-9, 7.0])) == 1.0)
    assert np.all(np.diff(O.meyer_aux(np.linspace(0, 1, 1001))) >= 0)


def test_b_support_symmetry_values():
    # eq:b: b symmetric, positive, supp b = [-4,-1] u [1,4], b(+-2) = 1.
    w = np.linspace(-6, 6, 24001)
    b = O.bump_b(w)
    assert np.array_equal(b, O.bump_b(-w))
    inside = (np.abs(w) > 1.0 + 1e-9) & (np.abs(w) < 4.0 - 1e-9)
    assert np.all(b[inside] > 0)
    assert np.all(np.abs(b[(np.abs(w) < 1.0) | (np.abs(w) > 4.0)]) == 0.0)
    assert abs(O.bump_b(4.0)) < 1e-16 and O.bump_b(1.0) == 0.0
    # b(1.5) = sin(pi/2 v(1/2)) = sin(pi/4)   (S:L46-49 derived)
    assert O.bump_b(1.5) == pytest.approx(math.sqrt(0.5), abs=1e-15)


def test_b_dyadic_partition_of_unity():
    # Lemma propertySumbj: sum_{j>=-1} b^2(2^-j w) = 1 for |w| >= 1,
    # and eq:OverlapPsi1: = sin^2(pi/2 v(2w-1)) on 1/2<|w|<1, 0 on |w|<=1/2.
    w = np.concatenate([np.linspace(1.0, 300.0, 50001), -np.linspace(1.0, 50.0, 3001)])
    s = sum(O.bump_b(2.0 ** (-j) * w) ** 2 for j in range(-1, 12))
    assert np.max(np.abs(s - 1.0)) < 1e-13
    w2 = np.linspace(0.5001, 0.9999, 2001)
    s2 = sum(O.bump_b(2.0 ** (-j) * w2) ** 2 for j in range(-1, 5))
    ref = np.sin(np.pi / 2 * (35 * (2 * w2 - 1) ** 4 - 84 * (2 * w2 - 1) ** 5
                              + 70 * (2 * w2 - 1) ** 6 - 20 * (2 * w2 - 1) ** 7)) ** 2
    assert np.max(np.abs(s2 - ref)) < 1e-13
    assert np.all(sum(O.bump_b(2.0 ** (-j) * np.linspace(0, 0.5, 101)) ** 2
                      for j in range(-1, 5)) == 0.0)


def test_psi1_composition_matches_closed_form():
    # eq:Psi1 composition sqrt(b^2(2w)+b^2(w)) against the piecewise form the
    # paper derives in Sec. 3.4: two different formulas of the paper.
    w = np.linspace(-5, 5, 40001)
    assert np.max(np.abs(O.psi1_hat(w) - O.psi1_hat_closed_form(w))) < 1e-15
    # Thm PropertyPsi1: supp = [-4,-1/2] u [1/2,4]
    assert np.all(O.psi1_hat(w[(np.abs(w) <= 0.5) | (np.abs(w) >= 4.0)]) < 1e-16)
    assert np.all(O.psi1_hat(w[(np.abs(w) > 0.5 + 1e-9) & (np.abs(w) < 4 - 1e-9)]) > 0)
    assert O.psi1_hat(0.75) == pytest.approx(math.sqrt(0.5), abs=1e-15)


def test_psi1_dyadic_sum():
    # Thm PropertyPsi1: sum_{j>=0} |psi1_hat(2^-2j w)|^2 = 1 for |w| > 1;
    # eq:OverlapPsi1_2: = sin^2(pi/2 v(2w-1)) on (1/2,1).
    w = np.linspace(1.0001, 4000.0, 80001)
    s = sum(O.psi1_hat(4.0 ** (-j) * w) ** 2 for j in range(0, 10))
    assert np.max(np.abs(s - 1.0)) < 1e-13
    w2 = np.linspace(0.501, 0.999, 999)
    s2 = sum(O.psi1_hat(4.0 ** (-j) * w2) ** 2 for j in range(0, 4))
    assert np.max(np.abs(s2 - np.sin(np.pi / 2 * O.meyer_aux(2 * w2 - 1)) ** 2)) < 1e-13


def test_psi1_truncated_sum_plateau():
    # Sec. 3.5.2: sum_{j=0}^{j0-1} psi1(2^-2j w)^2 = 1 on [1, 2^(2 j0 - 1)],
    # which is why X = 2^(2 j0 - 1).
    for j0 in range(1, 6):
        w = np.linspace(1.0, 2.0 ** (2 * j0 - 1), 20001)
        s = sum(O.psi1_hat(4.0 ** (-j) * w) ** 2 for j in range(j0))
        assert np.max(np.abs(s - 1.0)) < 1e-13, j0


def test_psi2_properties():
    # eq:Psi2: psi2(0)=1, psi2(+-1)=0, supp [-1,1], even.
    w = np.linspace(-3, 3, 30001)
    p = O.psi2_hat(w)
    assert np.array_equal(p, O.psi2_hat(-w))
    assert O.psi2_hat(0.0) == 1.0 and O.psi2_hat(1.0) == 0.0 and O.psi2_hat(-1.0) == 0.0
    assert np.all(p[np.abs(w) >= 1.0] == 0.0)
    # Lemma PropertyPsi2: psi2^2(w-1)+psi2^2(w)+psi2^2(w+1) = 1 on |w|<=1
    w1 = np.linspace(-1, 1, 20001)
    s = O.psi2_hat(w1 - 1) ** 2 + O.psi2_hat(w1) ** 2 + O.psi2_hat(w1 + 1) ** 2
    assert np.max(np.abs(s - 1.0)) < 1e-13
    # Thm PropertyPsi2: sum_{k=-2^j}^{2^j} psi2(k + 2^j w)^2 = 1 for |w|<=1
    for j in range(0, 5):
        K = 2 ** j
        s = sum(O.psi2_hat(k + K * w1) ** 2 for k in range(-K, K + 1))
        assert np.max(np.abs(s - 1.0)) < 1e-13, j


def test_scaling_matches_psi1():
    # eq:overlapPsi1Phi: |psi1(w)|^2 + |varphi(w)|^2 = 1 on [1/2, 1]
    w = np.linspace(0.5, 1.0, 10001)
    assert np.max(np.abs(O.psi1_hat(w) ** 2 + O.scaling_varphi(w) ** 2 - 1)) < 1e-13
    assert np.all(O.scaling_varphi(np.linspace(-0.5, 0.5, 101)) == 1.0)
    assert np.all(O.scaling_varphi(np.array([1.0, -1.0, 1.5])) == 0.0)


# ---------------------------------------------------------------- sizes and indexing

def test_j0_table():
    for lo, hi, j0 in _golden_rows("j0_table.txt"):
        for n in range(int(lo), int(hi) + 1):
            assert O.scales_for_size(n) == int(j0), n
    assert O.scales_for_size(4096) == 6
    with pytest.raises(ValueError):
        O.scales_for_size(3)


def test_eta_table_and_closed_form():
    for j0, eta in _golden_rows("eta_table.txt"):
        assert O.num_shearlets(int(j0)) == int(eta)
    for j0 in range(1, 9):
        assert O.num_shearlets(j0) == 2 ** (j0 + 2) - 3     # eq:numberOfScalesAndShears


def test_index_order():
    counts = {row[0]: int(row[1]) for row in _golden_rows("band_counts.txt")}
    j0 = 3
    table = [O.index_to_params(j0, i) for i in range(1, O.num_shearlets(j0) + 1)]
    assert table[0] == (O.KIND_S, 0, 0) and counts["lowpass"] == 1       # "i=1 for the low-pass"
    for j in range(j0):
        band = [t for t in table if t[0] != O.KIND_S and t[1] == j]
        if f"j{j}" in counts:
            assert len(band) == counts[f"j{j}"]
        assert len(band) == 2 ** (j + 2)
        K = 2 ** j
        assert band[0] == (O.KIND_H, j, 0)                               # "start in the horizontal position"
        assert band[1:K] == [(O.KIND_H, j, -k) for k in range(1, K)]     # k = -1 .. -2^j+1
        assert band[K] == (O.KIND_X, j, -K)                              # diagonal, slope 1
        assert band[K + 1:3 * K] == [(O.KIND_V, j, k) for k in range(-K + 1, K)]
        assert band[3 * K] == (O.KIND_X, j, K)
        # every (kind,j,k) of the frame in Thm discreteShearletFrame appears exactly once
        ks_h = sorted(t[2] for t in band if t[0] == O.KIND_H)
        assert ks_h == list(range(-K + 1, K))
    for i in range(1, len(table) + 1):
        assert O.params_to_index(j0, *table[i - 1]) == i
    with pytest.raises(IndexError):
        O.index_to_params(j0, 0)
    with pytest.raises(IndexError):
        O.params_to_index(j0, O.KIND_X, 1, 1)


def test_grid():
    # Delta = 1 if N = 2^(2 j0) + 1;  X = 2^(2 j0 - 1)
    axis, n_odd, X, d = O.frequency_grid(17)
    assert (n_odd, X, d) == (17, 8.0, 1.0) and axis[0] == -8 and axis[-1] == 8
    axis, n_odd, X, d = O.frequency_grid(64)
    assert (n_odd, X, d) == (65, 32.0, 1.0) and axis[32] == 0.0
    axis, n_odd, X, d = O.frequency_grid(512)
    assert (n_odd, X, d) == (513, 128.0, 0.5)
    for n in (5, 9, 33, 100, 1000):
        axis, n_odd, X, d = O.frequency_grid(n)
        assert 0.25 < d <= 1.0 and axis[0] == -X and axis[-1] == X    # 1/4 < Delta <= 1


# ---------------------------------------------------------------- spectra

@pytest.mark.parametrize("n", [4, 5, 8, 9, 16, 17, 32, 33, 64, 65, 128, 256])
def test_frame_tightness(n):
    # Thm discreteShearletFrame / Fig. frameTightness:
    # sum_i psi_i^2 = 1 at every grid point; the paper prints ~8e-15.
    psi = O.shearlet_spectra(n)
    dev = np.max(np.abs(np.sum(psi**2, axis=0) - 1.0))
    assert dev < 1e-13, dev


def test_frame_tightness_other_j0():
    # numOfScales option [reading A17]: tiling holds for any j0 because
    # X and Delta are derived from j0.
    for j0 in (1, 2, 3, 4):
        psi = O.shearlet_spectra(64, j0)
        assert psi.shape[0] == 2 ** (j0 + 2) - 3
        assert np.max(np.abs(np.sum(psi**2, axis=0) - 1.0)) < 1e-13


def test_spectra_odd_grid_even_and_supports():
    # odd N: every plane is point-symmetric psi(-w) = psi(w) (the grid is symmetric);
    # cone supports: h planes vanish off C^h, v planes off C^v.
    n, j0 = 65, 3
    axis, *_ = O.frequency_grid(n)
    w1, w2 = np.meshgrid(axis, axis)
    for i in range(1, O.num_shearlets(j0) + 1):
        p = O.shearlet_spectrum(n, i)
        assert np.array_equal(p, p[::-1, ::-1])
        kind, j, k = O.index_to_params(j0, i)
        if kind == O.KIND_H:
            assert np.all(p[np.abs(w2) >= np.abs(w1)] == 0.0)
        if kind == O.KIND_V:
            assert np.all(p[np.abs(w1) >= np.abs(w2)] == 0.0)


def test_even_n_is_delta_scaled_omega():
    # sampling psi(Delta * omega) on Omega gives the same spectra as the
    # cropped odd-grid construction of P:L2151-2153 [reading A4].
    n = 64
    axis, _, _, d = O.frequency_grid(n)
    om = np.arange(-n // 2, n // 2) * d
    assert np.array_equal(axis[:n], om)


def test_seam_value():
    # glued diagonal on the slope-1 diagonal w2 = w1 with k = -2^j equals
    # psi1(4^-j w1) * psi2(0) = psi1(4^-j w1) (frame proof's "= 1" underbrace).
    n, j0 = 64, 3
    axis, *_ = O.frequency_grid(n)
    for j in range(j0):
        i = O.params_to_index(j0, O.KIND_X, j, -2 ** j)
        p = O.shearlet_spectrum(n, i)
        for u in range(1, n // 2):
            c = n // 2 + u
            assert p[c, c] == pytest.approx(float(O.psi1_hat(4.0 ** (-j) * axis[c])), abs=1e-15)


# ---------------------------------------------------------------- DFTs and transform

@pytest.mark.parametrize("n", [4, 5, 8, 9, 16])
def test_dft_library_matches_direct(n):
    # P:L902-912 written out as double sums vs the library FFT step.
    rng = np.random.default_rng(n)
    f = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    assert np.max(np.abs(O.dft2_centred(f) - O.dft2_direct(f))) < 1e-12
    assert np.max(np.abs(O.idft2_centred(f) - O.idft2_direct(f))) < 1e-13
    assert np.max(np.abs(O.idft2_direct(O.dft2_direct(f)) - f)) < 1e-13


@pytest.mark.parametrize("n", [8, 9, 16])
def test_forward_fft_equals_direct(n):
    f = synth.uniform_image(n, 11)
    a = O.forward(f)
    b = O.forward(f, direct=True)
    assert np.max(np.abs(a - b)) < 1e-13


@pytest.mark.parametrize("n", [8, 9, 16])
def test_parseval_matrix_brute_force(n):
    # Parseval frame <=> U^H U = I, U built column by column with the
    # direct (no-FFT) transform.
    psi = O.shearlet_spectra(n)
    cols = []
    for m in range(n * n):
        e = np.zeros(n * n)
        e[m] = 1.0
        cols.append(O.forward(e.reshape(n, n), psi=psi, direct=True).ravel())
    u = np.stack(cols, axis=1)
    g = u.conj().T @ u
    assert np.max(np.abs(g - np.eye(n * n))) < 1e-13


@pytest.mark.parametrize("n", [32, 64, 65, 256])
def test_parseval_and_round_trip(n):
    # Parseval ||f||^2 = sum_i ||c_i||^2 and exactness (Fig. transformExactness,
    # ~2e-15 for a random image).
    f = synth.uniform_image(n, 100 + n)
    c = O.forward(f)
    rel = abs(np.sum(np.abs(c) ** 2) - np.sum(f**2)) / np.sum(f**2)
    assert rel < 1e-13
    rec = O.inverse(c)
    assert np.max(np.abs(rec.real - f)) < 1e-13
    assert np.max(np.abs(rec.imag)) < 1e-13
    exactness = float(_golden_rows("paper_accuracy.txt")[1][1])
    assert np.max(np.abs(rec.real - f)) < 50 * exactness


def test_complex_coefficients_even_n():
    # [reading A8] even N: finest-scale k != 0 planes carry a real imaginary part, and
    # dropping it breaks the round trip; odd N: coefficients are real.
    f = synth.uniform_image(64, 5)
    c = O.forward(f)
    assert np.max(np.abs(c.imag)) > 1e-3
    assert np.max(np.abs(O.inverse(c.real).real - f)) > 1e-3
    c_odd = O.forward(synth.uniform_image(65, 5))
    assert np.max(np.abs(c_odd.imag)) < 1e-13


def test_constant_image():
    # every shearlet spectrum vanishes at omega = 0 (supp psi1 excludes 0): only the
    # low-pass plane (i=1) is non-zero and it equals the constant.
    n = 32
    c = O.forward(np.full((n, n), 0.7))
    assert np.max(np.abs(c[0] - 0.7)) < 1e-13
    assert np.max(np.abs(c[1:])) < 1e-13


def test_shift_covariance():
    # each plane is a Fourier multiplier: translating f translates every plane
    # ("translates ... over the full grid", discrete t_m of eq:discrete_t).
    n = 64
    f = synth.uniform_image(n, 3)
    c = O.forward(f)
    cs = O.forward(np.roll(f, (5, -9), axis=(0, 1)))
    assert np.max(np.abs(cs - np.roll(c, (5, -9), axis=(1, 2)))) < 1e-13


def test_orientation():
    # A vertical line has its spectrum on omega_2 = 0: the horizontal-cone, k = 0 shearlet
    # of the finest scale carries the largest energy among the shearlet planes (Fig. 1 idea,
    # P:L42-55; axis reading A3).
    n = 64
    j0 = O.scales_for_size(n)
    c = O.forward(synth.vertical_line_image(n))
    energy = np.sum(np.abs(c) ** 2, axis=(1, 2))
    best = int(np.argmax(energy[1:])) + 2
    assert O.index_to_params(j0, best) == (O.KIND_H, j0 - 1, 0)


def test_single_plane_inverse():
    # inverse of a cube holding one plane c_i only: ifft2(psi_i^2 f_hat) (eq:inverseShearletTransform)
    n = 32
    f = synth.uniform_image(n, 8)
    psi = O.shearlet_spectra(n)
    c = O.forward(f, psi=psi)
    i = 9
    rec = O.inverse(c[i - 1:i], psi=psi, planes=[i])
    ref = np.fft.ifft2(np.fft.ifftshift(psi[i - 1] ** 2 * np.fft.fftshift(np.fft.fft2(f))))
    assert np.max(np.abs(rec - ref)) < 1e-13


@pytest.mark.parametrize("n", [16, 32, 64])
def test_adjoint_identity(n):
    # inverse = adjoint of forward: Re <T f, Z> = <f, Re T* Z> for real f
    # and an arbitrary complex cube Z (pins the inverse off the range of the forward).
    f = synth.uniform_image(n, 21)
    eta = O.num_shearlets(O.scales_for_size(n))
    z = synth.random_cube((eta, n, n), 22)
    lhs = np.real(np.sum(O.forward(f) * np.conj(z)))
    rhs = np.sum(f * O.inverse(z).real)
    assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs))


@pytest.mark.parametrize("n", [16, 32])
def test_imaginary_part_rank_two(n):
    # SURVEY 8(a) / DESIGN 6.2: for even n, Im c_i = (-1)^r G_i(m1) + (-1)^m1 H_i(r) (rank <= 2):
    # the compact coefficient format (real part + two n-vectors per plane) is lossless for
    # the forward's output.  Pinned here on the oracle's cube of a random image.
    f = synth.uniform_image(n, seed=11)
    c = O.forward(f)
    m = np.arange(n)
    sgn = (-1.0) ** m
    for i in range(c.shape[0]):
        y = c[i].imag
        # G, H from row 0 / column 0 up to the gauge (G + a(-1)^m1, H - a(-1)^r)
        g = y[0, :] - 0.0
        h = (y[:, 0] - sgn * g[0]) * sgn[0]
        rec = sgn[:, None] * g[None, :] + sgn[None, :] * h[:, None]
        assert np.max(np.abs(rec - y)) <= 1e-12 * max(1.0, np.max(np.abs(c[i])))
        assert np.linalg.matrix_rank(y, tol=1e-10 * max(1.0, np.max(np.abs(y)))) <= 2


# ---------------------------------------------------------------- smooth variant

@pytest.mark.parametrize("n", [8, 9, 32, 33, 64, 65, 256])
def test_smooth_frame_tightness(n):
    # Sec. smoothShearlets: Phi^2(w) + sum_j Psi1^2(4^-j w) telescopes to
    # Phi^2(4^-j0 w) = 1 on the grid, and the psi2 shears tile each cone as before, so the
    # smooth system is again a Parseval frame: sum_i psi_i^2 = 1 at every grid point.
    psi = O.shearlet_spectra(n, variant="smooth")
    assert psi.shape[0] == O.num_shearlets(O.scales_for_size(n))
    dev = np.max(np.abs(np.sum(psi**2, axis=0) - 1.0))
    assert dev < 1e-13, dev


def test_smooth_psi1_support_and_axis():
    # Psi1 is supported in [-4,4]^2 minus [-1/2,1/2]^2.  On an axis Phi = varphi, so
    # Psi1(w1, 0)^2 = varphi^2(w1/4) - varphi^2(w1), which the partition of unity
    # varphi^2 + sum_j psi1^2(4^-j .) = 1 makes psi1_hat(w1)^2: the
    # smooth corona function restricted to an axis is the classic radial function.
    g = np.linspace(-5, 5, 401)
    w1, w2 = np.meshgrid(g, g)
    p = O.smooth_psi1(w1, w2)
    m = np.maximum(np.abs(w1), np.abs(w2))
    assert np.all(p[(m <= 0.5) | (m >= 4.0)] == 0.0)
    assert np.all(p[(m > 0.55) & (m < 3.9)] > 0.0)
    x = np.linspace(-5, 5, 2001)
    # the printed difference evaluated in float64 alone is only sqrt(eps)-accurate next to
    # |w| = 1/2; the oracle's 40-digit re-evaluation of the same formula is exact to rounding
    assert np.max(np.abs(O.smooth_psi1(x, 0.0 * x, precise=False) - O.psi1_hat(x))) > 1e-12
    assert np.max(np.abs(O.smooth_psi1(x, 0.0 * x) - O.psi1_hat(x))) < 1e-13
    assert np.max(np.abs(O.smooth_psi1(x, 0.0 * x) ** 2 - O.psi1_hat(x) ** 2)) < 1e-14
    # tensor scaling function: 1 on [-1/2,1/2]^2, 0 once a coordinate reaches 1, symmetric
    assert np.all(O.tensor_scaling_Phi(w1, w2)[m <= 0.5] == 1.0)
    assert np.all(O.tensor_scaling_Phi(w1, w2)[m >= 1.0] == 0.0)
    assert np.array_equal(O.tensor_scaling_Phi(w1, w2), O.tensor_scaling_Phi(w2, w1))


def test_smooth_psi1_off_axis_closed_form():
    # Off the axes, with both |w_i| < 1: Phi(w/4) = 1 there (|w_i|/4 < 1/4), so eq:newPsi1 is
    # sqrt(1 - varphi^2(w1) varphi^2(w2)).  With varphi^2 = 1 - s_i, s_i = sin^2(pi/2 v(2|w_i|-1))
    # on 1/2 < |w_i| < 1, 1 - varphi1^2 varphi2^2 = s1 + s2 - s1 s2: a sum that does
    # not cancel, evaluated here independently of the printed difference.
    g = np.concatenate([np.linspace(0.5, 0.52, 401), np.linspace(0.52, 0.999, 300)])
    w1, w2 = np.meshgrid(g, g[::7])
    s = lambda w: np.where(np.abs(w) > 0.5, np.sin(np.pi / 2 * O.meyer_aux(2 * np.abs(w) - 1)) ** 2, 0.0)
    s1, s2 = s(w1), s(w2)
    ref = np.sqrt(s1 + s2 - s1 * s2)
    assert np.max(np.abs(O.smooth_psi1(w1, w2) - ref)) < 1e-13
    assert np.max(np.abs(O.smooth_psi1(-w1, w2) - ref)) < 1e-13


@pytest.mark.parametrize("variant", ["classic", "smooth"])
@pytest.mark.parametrize("n", [16, 32, 33, 64])
def test_forward_plane_is_a_plane_of_forward(n, variant):
    # forward_plane (the per-plane form the large-n parity tests use) is plane i of the whole
    # transform eq:shearletTransform, for every flat index i, both systems, even
    # and odd n; forward itself is pinned by the direct DFT, Parseval and the round trip above.
    f = synth.make_batch(1, n=n)[0]
    full = O.forward(f, variant=variant)
    f_hat = O.dft2_centred(f)
    for i in range(1, full.shape[0] + 1):
        a = O.forward_plane(f, i, variant=variant)
        b = O.forward_plane(f, i, f_hat=f_hat, variant=variant)
        assert np.max(np.abs(a - full[i - 1])) <= 1e-15 * max(1.0, np.max(np.abs(full))), i
        assert np.array_equal(a, b)
    with pytest.raises(IndexError):
        O.forward_plane(f, full.shape[0] + 1, variant=variant)


def test_smooth_equals_classic_near_the_axis():
    # In the horizontal cone at scale j, where |4^-j w2| <= 1/2 the second factor of Phi is 1 at
    # both dilations, so Psi1(4^-j w) = psi1_hat(4^-j w1) and the smooth cone shearlet equals the
    # classic one (eq:newPsi1 vs eq:Psi1); the two systems differ only away from the axes.
    n = 128
    j0 = O.scales_for_size(n)
    axis, *_ = O.frequency_grid(n, j0)
    w1, w2 = np.meshgrid(axis[:n], axis[:n])
    differs = 0
    for i in range(2, O.num_shearlets(j0) + 1):
        kind, j, k = O.index_to_params(j0, i)
        if kind != O.KIND_H:
            continue
        a = O.shearlet_spectrum(n, i, j0)
        b = O.shearlet_spectrum(n, i, j0, variant="smooth")
        near = np.abs(w2) * 4.0 ** (-j) <= 0.5
        assert np.max(np.abs(a[near] - b[near])) < 1e-7
        differs += int(np.max(np.abs(a - b)) > 1e-3)
    assert differs > 0


@pytest.mark.parametrize("n", [16, 33])
def test_smooth_round_trip_and_parseval(n):
    # Parseval frame: ||SH f||^2 = ||f||^2 and the adjoint inverts the transform.
    f = synth.make_batch(1, n=n)[0]
    c = O.forward(f, variant="smooth")
    assert abs(np.sum(np.abs(c) ** 2) - np.sum(f**2)) < 1e-10 * np.sum(f**2)
    rec = O.inverse(c, variant="smooth")
    assert np.max(np.abs(rec.real - f)) < 1e-11 * np.max(np.abs(f))


def test_unknown_variant_rejected():
    with pytest.raises(ValueError):
        O.shearlet_spectrum(16, 2, variant="bogus")


# ---------------------------------------------------------------- user-supplied spectra

def test_frame_tightness_check():
    # sum(abs(Psi).^2,3) - 1 is ~0 for a Parseval system (the built-in one: the
    # paper's Fig. frameTightness level) and exactly 3 when every spectrum is doubled.
    psi = O.shearlet_spectra(32)
    assert O.frame_tightness(psi) < 1e-13
    assert abs(O.frame_tightness(2.0 * psi) - 3.0) < 1e-12
    assert O.frame_tightness(synth.random_spectra(16, 5, 1)) < 1e-14
    assert O.frame_tightness(synth.random_spectra(16, 5, 1, parseval=False)) > 1e-2


@pytest.mark.parametrize("n,eta", [(8, 3), (16, 7)])
def test_user_spectra_parseval_and_brute_force(n, eta):
    # The transform with precomputed spectra: for any Parseval system the adjoint
    # inverts it (P:L1730-1764 with sum_i psi_i^2 = 1) and energy is kept; and one coefficient of
    # one plane against the double sum of its definition (eq:shearletTransform written out,
    # brute force: c_i(x) = 1/N^2 sum_w psi_i(w) f_hat(w) e^{+2 pi i <w, x>/N}).
    psi = synth.random_spectra(n, eta, 11)
    f = synth.uniform_image(n, 5)
    c = O.forward(f, psi=psi)
    assert abs(np.sum(np.abs(c) ** 2) - np.sum(f**2)) < 1e-12 * np.sum(f**2)
    rec = O.inverse(c, psi=psi)
    assert np.max(np.abs(rec - f)) < 1e-12 * np.max(np.abs(f))
    h = n // 2
    u = np.arange(n) - h
    x = np.arange(n) - h
    fh = np.array([[sum(f[r, m] * np.exp(-2j * np.pi * (a1 * (m - h) + a2 * (r - h)) / n)
                        for r in range(n) for m in range(n)) for a1 in u] for a2 in u])
    for i in (0, eta - 1):
        for (r, m) in ((0, 0), (3, n - 1), (h, 1)):
            val = sum(psi[i, p, q] * fh[p, q] * np.exp(2j * np.pi * (u[q] * x[m] + u[p] * x[r]) / n)
                      for p in range(n) for q in range(n)) / n**2
            assert abs(val - c[i, r, m]) < 1e-12, (i, r, m)


def test_oracle_pool_matches_oracle():
    # the tests' parallel driver of the oracle (tests/oracle_pool.py) returns exactly what the
    # oracle's own functions return (same terms, summed in the same plane order)
    import oracle_pool as OP
    n = 32
    f = synth.make_batch(1, n=n)[0]
    planes = [0, 3, 7, 12]
    got = OP.forward_planes(f, planes)
    for i in planes:
        assert np.array_equal(got[i], O.forward_plane(f, i + 1))
    z = synth.random_cube((len(planes), n, n), 5)
    assert np.array_equal(OP.inverse(z, planes), O.inverse(z, planes=[i + 1 for i in planes]))
