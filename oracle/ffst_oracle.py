"""FFST oracle: a plain, slow, float64 CPU implementation of the Fast Finite
Shearlet Transform of arxiv 1202.1773 ("PAPER.md"), written from the paper.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
execute this module: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use it.  It
shares no code with the CUDA path (``paper_1202_1773_b200/``), and the CUDA
path never imports it.

Citation keys: ``P:Lnnn`` is a line of PAPER.md (section / equation named
beside it).  Every function follows the passage it cites, in the paper's
notation and order.  Readings of places where the paper is silent, ambiguous
or garbled are the ones listed in DESIGN.md ("Readings of the paper") and are
marked ``[reading Ax]`` below.

Conventions:
  * an image ``f`` is ``f[m2, m1]`` (rows = m2, columns = m1);
  * spectra and centred DFTs are ``X[omega2, omega1]`` with the centred index
    set Omega = {-floor(N/2) .. ceil(N/2)-1}, i.e. numpy's
    ``fftshift`` order;
  * forward DFT unnormalised, inverse with 1/N^2.

Parity: every function here is pinned by ``tests/test_oracle_pins.py``
against values, closed forms and identities the paper fixes (no function is
"parity unpinned"; the plane *order* inside a band beyond its counts is a
labelling convention, [reading A1]).
"""
from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

__all__ = [
    "meyer_aux", "bump_b", "psi1_hat", "psi1_hat_closed_form", "psi2_hat",
    "scaling_varphi", "scales_for_size", "num_shearlets", "index_to_params",
    "params_to_index", "frequency_grid", "shearlet_spectrum", "shearlet_spectra",
    "dft2_centred", "idft2_centred", "dft2_direct", "idft2_direct",
    "forward", "forward_plane", "inverse", "tensor_scaling_Phi", "smooth_psi1", "frame_tightness", "KIND_S", "KIND_H", "KIND_V", "KIND_X",
]

KIND_S, KIND_H, KIND_V, KIND_X = 0, 1, 2, 3   # low-pass, horizontal, vertical, seam ("h x v")


# ---------------------------------------------------------------------------
# 2.1  Window functions
# ---------------------------------------------------------------------------

def meyer_aux(x):
    """Meyer's auxiliary function v, eq:v (Sec. 2.1):
    0 for x<0;  35x^4 - 84x^5 + 70x^6 - 20x^7 for 0<=x<=1;  1 for x>1."""
    x = np.asarray(x, dtype=np.float64)
    x2 = x * x                      # the monomials as products (numpy's generic pow is ~10x slower)
    x4 = x2 * x2
    x5, x6 = x4 * x, x4 * x2
    x7 = x6 * x
    poly = 35.0 * x4 - 84.0 * x5 + 70.0 * x6 - 20.0 * x7
    return np.where(x < 0.0, 0.0, np.where(x > 1.0, 1.0, poly))


def bump_b(omega):
    """The function b, eq:b (Sec. 2.1):
    sin(pi/2 v(|w|-1)) for 1<=|w|<=2;  cos(pi/2 v(|w|/2-1)) for 2<|w|<=4;  0 otherwise."""
    a = np.abs(np.asarray(omega, dtype=np.float64))
    rising = np.sin(np.pi / 2.0 * meyer_aux(a - 1.0))
    falling = np.cos(np.pi / 2.0 * meyer_aux(a / 2.0 - 1.0))
    return np.where((a >= 1.0) & (a <= 2.0), rising,
                    np.where((a > 2.0) & (a <= 4.0), falling, 0.0))


def psi1_hat(omega):
    """Radial band-pass, eq:Psi1: psi1_hat(w) = sqrt(b^2(2w) + b^2(w))."""
    omega = np.asarray(omega, dtype=np.float64)
    return np.sqrt(bump_b(2.0 * omega) ** 2 + bump_b(omega) ** 2)


def psi1_hat_closed_form(omega):
    """The piecewise form of psi1_hat the paper derives in Sec. 3.4:
    0 (|w|<=1/2), sin(pi/2 v(2|w|-1)) (1/2<|w|<1), 1 (1<=|w|<=2),
    cos(pi/2 v(|w|/2-1)) (2<|w|<4), 0 (|w|>=4).  Used only as a pin of psi1_hat."""
    a = np.abs(np.asarray(omega, dtype=np.float64))
    return np.select(
        [a <= 0.5, a < 1.0, a <= 2.0, a < 4.0],
        [0.0, np.sin(np.pi / 2.0 * meyer_aux(2.0 * a - 1.0)), 1.0,
         np.cos(np.pi / 2.0 * meyer_aux(a / 2.0 - 1.0))],
        default=0.0)


def psi2_hat(omega):
    """Shear window, eq:Psi2: sqrt(v(1+w)) for w<=0, sqrt(v(1-w)) for w>0."""
    w = np.asarray(omega, dtype=np.float64)
    return np.where(w <= 0.0, np.sqrt(meyer_aux(1.0 + w)), np.sqrt(meyer_aux(1.0 - w)))


def scaling_varphi(omega):
    """Mother scaling function varphi (Sec. 2.4):
    1 for |w|<=1/2;  cos(pi/2 v(2|w|-1)) for 1/2<|w|<1;  0 otherwise."""
    a = np.abs(np.asarray(omega, dtype=np.float64))
    return np.where(a <= 0.5, 1.0,
                    np.where(a < 1.0, np.cos(np.pi / 2.0 * meyer_aux(2.0 * a - 1.0)), 0.0))


def tensor_scaling_Phi(omega1, omega2):
    """Tensor-product scaling function, eq:Phi: Phi(w) = varphi(w1) varphi(w2).
    The low-pass of the smooth construction (Sec. smoothShearlets)."""
    return scaling_varphi(omega1) * scaling_varphi(omega2)


def smooth_psi1(omega1, omega2, precise: bool = True):
    """eq:newPsi1: Psi1(w) = sqrt(Phi^2(w/4) - Phi^2(w)), written out as printed
    (clipped at 0 against rounding).  Supported in [-4,4]^2 minus [-1/2,1/2]^2.

    In float64 the printed difference of two squares cancels where both are close to 1 (just
    outside |w_i| = 1/2, where varphi = 1 - O(v^2)): the square root of an O(eps) difference is
    then good to only ~sqrt(eps) absolute.  ``precise`` re-evaluates the same printed formula --
    v, varphi, Phi, the difference and the root -- in 40-digit arithmetic (mpmath) wherever the
    float64 difference is a cancellation below 1e-4 (Phi(w) > 0 and not both |w_i| <= 1/2, where
    the exact value is 0), so the result is correct to ~1e-14 absolute everywhere [reading A19]."""
    omega1 = np.asarray(omega1, dtype=np.float64)
    omega2 = np.asarray(omega2, dtype=np.float64)
    phi_w = tensor_scaling_Phi(omega1, omega2)
    d = tensor_scaling_Phi(omega1 / 4.0, omega2 / 4.0) ** 2 - phi_w ** 2
    out = np.sqrt(np.maximum(d, 0.0))
    if not precise:
        return out
    w1b, w2b = np.broadcast_arrays(omega1, omega2)
    out = np.array(np.broadcast_to(out, w1b.shape), dtype=np.float64)
    small = np.broadcast_to((d < 1e-4) & (phi_w > 0.0) & (np.maximum(np.abs(omega1), np.abs(omega2)) > 0.5),
                            w1b.shape)
    if np.any(small):
        # Psi1 depends on (|w1|, |w2|) only: evaluate each distinct pair once
        a1 = np.abs(w1b[small])
        a2 = np.abs(w2b[small])
        pairs = np.stack([a1, a2], axis=1)
        uniq, inv = np.unique(pairs, axis=0, return_inverse=True)
        vals = np.array([_smooth_psi1_mp(float(x), float(y)) for x, y in uniq], dtype=np.float64)
        out[small] = vals[np.asarray(inv).reshape(-1)]
    return out


def _smooth_psi1_mp(a1: float, a2: float) -> float:
    """eq:newPsi1 at one point, every step of the printed formula in 40-digit arithmetic:
    v (eq:v), varphi, Phi = varphi(w1) varphi(w2) (eq:Phi),
    sqrt(Phi^2(w/4) - Phi^2(w)).  The inputs are the exact float64 grid values."""
    import mpmath as mp
    with mp.workdps(40):
        def v(x):
            if x < 0:
                return mp.mpf(0)
            if x > 1:
                return mp.mpf(1)
            return 35 * x**4 - 84 * x**5 + 70 * x**6 - 20 * x**7

        def varphi(w):
            a = abs(w)
            if a <= mp.mpf(1) / 2:
                return mp.mpf(1)
            if a < 1:
                return mp.cos(mp.pi / 2 * v(2 * a - 1))
            return mp.mpf(0)

        x1, x2 = mp.mpf(a1), mp.mpf(a2)
        big = (varphi(x1 / 4) * varphi(x2 / 4)) ** 2
        small = (varphi(x1) * varphi(x2)) ** 2
        d = big - small
        return float(mp.sqrt(d)) if d > 0 else 0.0


# ---------------------------------------------------------------------------
# 3.5.1 / 3.5.2  Scales, indexing, grid
# ---------------------------------------------------------------------------

def scales_for_size(n: int) -> int:
    """j0 = floor(1/2 log2 N), computed with the integer
    bit length (no floating log2).  N < 4 has no scale (table starts at 4)."""
    n = int(n)
    if n < 4:
        raise ValueError(f"image size {n} < 4: no scale fits (P:L2163-2168)")
    return (n.bit_length() - 1) // 2


def num_shearlets(j0: int) -> int:
    """eta = 1 + sum_{j<j0} 2^(j+2) = 2^(j0+2) - 3, eq:numberOfScalesAndShears."""
    return 1 + sum(2 ** (j + 2) for j in range(int(j0)))


@lru_cache(maxsize=None)
def _index_table(j0: int):
    """Flat index order of Sec. 3.5.1: i=1 low-pass; then per band
    j=0..j0-1 the lines rotate counter-clockwise: (h,0), (h,-1..-(2^j-1)),
    (x,-2^j), (v,-2^j+1..2^j-1), (x,+2^j), (h, 2^j-1..1) [reading A1]."""
    table = [(KIND_S, 0, 0)]
    for j in range(j0):
        K = 2 ** j
        band = [(KIND_H, j, 0)]
        band += [(KIND_H, j, k) for k in range(-1, -K, -1)]
        band += [(KIND_X, j, -K)]
        band += [(KIND_V, j, k) for k in range(-K + 1, K)]
        band += [(KIND_X, j, K)]
        band += [(KIND_H, j, k) for k in range(K - 1, 0, -1)]
        table += band
    return tuple(table)


def index_to_params(j0: int, i: int):
    """Flat 1-based index i -> (kind, j, k) (helper/shearletScaleShear)."""
    table = _index_table(int(j0))
    if not 1 <= i <= len(table):
        raise IndexError(f"index {i} outside 1..{len(table)}")
    return table[i - 1]


def params_to_index(j0: int, kind: int, j: int, k: int) -> int:
    """Inverse of index_to_params (1-based)."""
    try:
        return _index_table(int(j0)).index((kind, j, k)) + 1
    except ValueError:
        raise IndexError(f"no shearlet ({kind},{j},{k}) for j0={j0}") from None


def frequency_grid(n: int, j0: int | None = None):
    """The lattice Xi of Sec. 3.5.2.

    N_odd = N if N is odd, else N+1; X = 2^(2 j0 - 1);
    Delta = 2^(2 j0) / (N_odd - 1); axis = -X .. X in N_odd points.
    Returns (axis, N_odd, X, Delta); for even N the caller drops the last
    row and column after computing the spectra."""
    if j0 is None:
        j0 = scales_for_size(n)
    n_odd = n if n % 2 == 1 else n + 1
    big_x = 2.0 ** (2 * j0 - 1)
    delta = 2.0 ** (2 * j0) / (n_odd - 1)
    half = (n_odd - 1) // 2
    axis = delta * np.arange(-half, half + 1, dtype=np.float64)
    return axis, n_odd, big_x, delta


# ---------------------------------------------------------------------------
# 2.3 / 3.1  Spectra on the grid
# ---------------------------------------------------------------------------

def _cone_shearlet(omega_a, omega_b, j, k):
    """psi_hat(4^-j w_a, 4^-j k w_a + 2^-j w_b) = psi1_hat(4^-j w_a) psi2_hat(2^j w_b/w_a + k)
    (eq:horizontalShearlet P:L607-615); 0 where w_a = 0 [reading A5]."""
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(omega_a != 0.0, omega_b / np.where(omega_a != 0.0, omega_a, 1.0), 0.0)
        value = psi1_hat(4.0 ** (-j) * omega_a) * psi2_hat(2.0 ** j * ratio + k)
    return np.where(omega_a != 0.0, value, 0.0)


def _smooth_cone_shearlet(omega_a, omega_b, j, k):
    """Smooth shearlet eq:smoothPsi at scale j, shear k:
    Psi1(4^-j w_a, 4^-j w_b) psi2_hat(2^j w_b/w_a + k) -- the corona function dilated
    isotropically so that sum_j Psi1^2(4^-j w) telescopes [reading A18];
    0 where w_a = 0 [reading A5]."""
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(omega_a != 0.0, omega_b / np.where(omega_a != 0.0, omega_a, 1.0), 0.0)
        value = smooth_psi1(4.0 ** (-j) * omega_a, 4.0 ** (-j) * omega_b) * psi2_hat(2.0 ** j * ratio + k)
    return np.where(omega_a != 0.0, value, 0.0)


def _spectrum_on_grid(w1, w2, kind, j, k, variant="classic"):
    """One spectrum psi_hat_{j,k,0}^kappa on the meshgrid (w1 = omega_1 columns,
    w2 = omega_2 rows), eq:shearletTransform's four cases.  variant "smooth":
    the construction of Sec. smoothShearlets: low-pass Phi (eq:Phi), cone
    shearlets from Psi1 (eq:newPsi1, eq:smoothPsi); cones and seam gluing unchanged."""
    a1, a2 = np.abs(w1), np.abs(w2)
    if variant == "smooth":
        if kind == KIND_S:
            return tensor_scaling_Phi(w1, w2)
        cone = _smooth_cone_shearlet
    elif variant == "classic":
        cone = _cone_shearlet
    else:
        raise ValueError(f"unknown variant {variant}")
    if kind == KIND_S:
        # eq:phi: varphi(w1) on |w1|<1, |w2|<=|w1|; varphi(w2) on |w2|<1, |w1|<|w2|
        return np.where((a1 < 1.0) & (a2 <= a1), scaling_varphi(w1),
                        np.where((a2 < 1.0) & (a1 < a2), scaling_varphi(w2), 0.0))
    chi_h = (a1 >= 0.5) & (a2 < a1)                    # C^h
    chi_v = (a2 >= 0.5) & (a2 > a1)                    # C^v
    chi_x = (a1 >= 0.5) & (a2 >= 0.5) & (a1 == a2)     # C^x, the seam [reading A6]
    if kind == KIND_H:                                 # eq:horizontalShearlet
        return cone(w1, w2, j, k) * chi_h
    if kind == KIND_V:                                 # eq:verticalShearlet
        return cone(w2, w1, j, k) * chi_v
    if kind == KIND_X:                                 # glued h + v + x, |k| = 2^j
        horizontal = cone(w1, w2, j, k)
        return (horizontal * chi_h + cone(w2, w1, j, k) * chi_v
                + horizontal * chi_x)                  # seam uses the horizontal formula (eq:seamlineShearlet)
    raise ValueError(f"unknown kind {kind}")


def shearlet_spectrum(n: int, i: int, j0: int | None = None, variant: str = "classic"):
    """Spectrum of flat index i (1-based) on the N x N centred grid, float64.

    Evaluated on the odd lattice Xi of Sec. 3.5.2; for even N the last row and
    column are dropped [reading A4].  Rows = omega_2, columns =
    omega_1 [reading A3]."""
    if j0 is None:
        j0 = scales_for_size(n)
    axis, n_odd, _, _ = frequency_grid(n, j0)
    w1, w2 = np.meshgrid(axis, axis)          # w1 varies along columns, w2 along rows
    kind, j, k = index_to_params(j0, i)
    spec = _spectrum_on_grid(w1, w2, kind, j, k, variant)
    return spec[:n, :n]


def shearlet_spectra(n: int, j0: int | None = None, variant: str = "classic"):
    """All eta spectra, shape (eta, N, N) ("Psi"); variant "classic"
    (meyerShearletSpect) or "smooth" (meyerNewShearletSpect)."""
    if j0 is None:
        j0 = scales_for_size(n)
    return np.stack([shearlet_spectrum(n, i, j0, variant) for i in range(1, num_shearlets(j0) + 1)])


# ---------------------------------------------------------------------------
# 3.1  DFTs
# ---------------------------------------------------------------------------

def dft2_centred(f):
    """f_hat(omega) = sum_m f(m) e^{-2 pi i (w1 m1 + w2 m2)/N}, omega in Omega (centred),
    P:L902-907.  numpy.fft (a library FFT) is the step; fftshift maps bins to Omega."""
    return np.fft.fftshift(np.fft.fft2(f, axes=(-2, -1)), axes=(-2, -1))


def idft2_centred(g):
    """f(m) = 1/N^2 sum_{omega in Omega} g(omega) e^{+2 pi i <omega, m/N>}."""
    return np.fft.ifft2(np.fft.ifftshift(g, axes=(-2, -1)), axes=(-2, -1))


def _omega(n):
    return np.arange(-(n // 2), (n + 1) // 2)


def dft2_direct(f):
    """The same DFT written out as the double sum of P:L902-907 (O(N^4)); pins dft2_centred."""
    n = f.shape[-1]
    om, m = _omega(n), np.arange(n)
    e = np.exp(-2j * np.pi * np.outer(om, m) / n)        # e[omega, m]
    return e @ f @ e.T                                   # rows: omega_2 <- m2, cols: omega_1 <- m1


def idft2_direct(g):
    """Direct inverse double sum of P:L908-912."""
    n = g.shape[-1]
    om, m = _omega(n), np.arange(n)
    e = np.exp(2j * np.pi * np.outer(m, om) / n)         # e[m, omega]
    return (e @ g @ e.T) / (n * n)


def frame_tightness(psi):
    """The Parseval check of P:L2219-2220 for any spectra set (built-in or user-supplied,
    P:L2209-2217): max over the grid of |sum_i psi_i^2 - 1| ("sum(abs(Psi).^2,3)-1")."""
    psi = np.asarray(psi, dtype=np.float64)
    return float(np.max(np.abs(np.sum(np.abs(psi) ** 2, axis=0) - 1.0)))


# ---------------------------------------------------------------------------
# 3.1 / 3.3  Forward and inverse transform
# ---------------------------------------------------------------------------

def forward(f, psi=None, j0: int | None = None, direct: bool = False, variant: str = "classic"):
    """Discrete shearlet transform, eq:shearletTransform:
    SH(f)(i) = ifft2(psi_hat_i * f_hat), one complex N x N plane per index i
    [reading A8: coefficients are complex].  Returns shape (eta, N, N) complex."""
    f = np.asarray(f, dtype=np.float64)
    n = f.shape[-1]
    if psi is None:
        psi = shearlet_spectra(n, j0, variant)
    dft, idft = (dft2_direct, idft2_direct) if direct else (dft2_centred, idft2_centred)
    f_hat = dft(f)
    return np.stack([idft(p * f_hat) for p in psi])


def forward_plane(f, i: int, j0: int | None = None, f_hat=None, variant: str = "classic"):
    """One plane of the forward transform (flat index i, 1-based), for sampled
    parity at sizes where the whole cube does not fit the host."""
    f = np.asarray(f, dtype=np.float64)
    n = f.shape[-1]
    if f_hat is None:
        f_hat = dft2_centred(f)
    return idft2_centred(shearlet_spectrum(n, i, j0, variant) * f_hat)


def inverse(coeffs, psi=None, j0: int | None = None, direct: bool = False, planes=None,
            variant: str = "classic"):
    """Inverse transform, eq:inverseShearletTransform:
    f_hat = sum_i fft2(c_i) * psi_hat_i;  f = ifft2(f_hat).

    Returns the complex ifft2 (the paper's literal result); the real-linear
    adjoint of ``forward`` is its real part [reading A9].  ``planes`` (1-based
    indices) restricts the sum to those planes (coeffs then holds only them)."""
    coeffs = np.asarray(coeffs, dtype=np.complex128)
    n = coeffs.shape[-1]
    if j0 is None:
        j0 = scales_for_size(n)
    if planes is None:   # every plane of the system (a user Psi has len(psi) planes)
        planes = range(1, (len(psi) if psi is not None else num_shearlets(j0)) + 1)
    dft, idft = (dft2_direct, idft2_direct) if direct else (dft2_centred, idft2_centred)
    acc = np.zeros((n, n), dtype=np.complex128)
    for slot, i in enumerate(planes):
        p = psi[i - 1] if psi is not None else shearlet_spectrum(n, i, j0, variant)
        acc += dft(coeffs[slot]) * p
    return idft(acc)
