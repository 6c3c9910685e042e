"""Parallel evaluation of the float64 oracle for the large-n parity tests (test infrastructure).

The oracle is plain single-threaded numpy; at n = 1024 / 4096 one plane costs seconds, so the
tests that compare many planes spread the oracle calls over host cores with a spawned process
pool (workers import only numpy, synth and the oracle).  Nothing here computes anything itself.
"""
from __future__ import annotations

import os

import numpy as np

_CACHE = {}


def _workers(n: int) -> int:
    per = 40 * n * n + (256 << 20)                      # a few float64 / complex128 planes per call
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    return max(1, min(os.cpu_count() or 1, 32, int(0.6 * avail // per)))


def _init(x64):
    import oracle as O
    _CACHE.clear()
    _CACHE["x"] = x64
    _CACHE["f_hat"] = O.dft2_centred(x64) if x64 is not None else None


def _forward_plane(args):
    i, variant = args
    import oracle as O
    return i, O.forward_plane(_CACHE["x"], i + 1, f_hat=_CACHE["f_hat"], variant=variant)


def _inverse_term(args):
    """psi_i * DFT2(z_i) for one plane (the summand of eq:inverseShearletTransform)."""
    i, z, variant = args
    import oracle as O
    n = z.shape[-1]
    return O.dft2_centred(z) * O.shearlet_spectrum(n, i + 1, variant=variant)


def forward_planes(x64, planes, variant="classic"):
    """{i: oracle.forward_plane(x64, i + 1)} for 0-based planes i."""
    import multiprocessing as mp
    n = x64.shape[-1]
    with mp.get_context("spawn").Pool(min(_workers(n), len(planes)), initializer=_init, initargs=(x64,)) as pool:
        return dict(pool.map(_forward_plane, [(i, variant) for i in planes], chunksize=1))


def inverse(z_planes, planes, variant="classic"):
    """oracle.inverse restricted to `planes` (0-based; z_planes[k] is plane planes[k]): the sum
    over the planes of psi_i * DFT2(z_i), then the inverse DFT -- the terms in parallel, summed in
    plane order."""
    import multiprocessing as mp
    import oracle as O
    n = z_planes.shape[-1]
    with mp.get_context("spawn").Pool(min(_workers(n), len(planes)), initializer=_init, initargs=(None,)) as pool:
        terms = pool.map(_inverse_term, [(i, np.asarray(z, dtype=np.complex128), variant)
                                         for i, z in zip(planes, z_planes)], chunksize=1)
    acc = np.zeros((n, n), dtype=np.complex128)
    for t in terms:
        acc += t
    return O.idft2_centred(acc)
