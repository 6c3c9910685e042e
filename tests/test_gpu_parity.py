"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on
the same seeded inputs.

Metric (reading A15, BASELINE.json tolerance): per-plane normwise
relative error max|gpu - oracle| / max|oracle|, worst plane, must be <= 1e-4
in float32 and <= 1e-10 in float64; the same on reconstructed images.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth

import oracle_pool as OP  # noqa: E402  (tests/oracle_pool.py)

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.float64: 1e-10}


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1202_1773_b200 as mod
    return mod


def plane_err(g, o, floor_scale=1.0):
    # reading A15: normwise per plane; a plane whose oracle values are zero up to rounding (e.g.
    # cos(pi/2) = 6e-17 at a band edge, reading A12) is compared in absolute terms, / max|f|
    g = np.asarray(g)
    o = np.asarray(o)
    num = np.max(np.abs(g - o), axis=(-2, -1))
    den = np.max(np.abs(o), axis=(-2, -1))
    small = den < 1e-12 * floor_scale
    return np.where(small, num / floor_scale, num / np.where(small, 1.0, den))


def images(cid, batch, n, dtype):
    x = synth.make_batch(cid, batch=batch, n=n)
    xt = torch.from_numpy(x).to(dtype)
    return xt, xt.double().numpy()          # the oracle consumes the cast values


# ------------------------------------------------------------------ spectra

@pytest.mark.parametrize("n,dtype", [(64, torch.float64), (256, torch.float32), (16, torch.float64),
                                     (4, torch.float64), (512, torch.float32)])
def test_spectra_match_oracle(F, n, dtype):
    plan = F.Plan(n, 1, dtype)
    psi = plan.spectra(centred=True).cpu().double().numpy()
    ref = O.shearlet_spectra(n)
    tol = 1e-13 if dtype == torch.float64 else 2e-6
    assert np.max(np.abs(psi - ref)) < tol
    # frame tightness of the on-the-fly window (Fig. frameTightness)
    assert np.max(np.abs(np.sum(psi**2, axis=0) - 1.0)) < (1e-13 if dtype == torch.float64 else 1e-5)


# ------------------------------------------------------------------ forward / inverse, small sizes

@pytest.mark.parametrize("tiny", ["1", "0"])
@pytest.mark.parametrize("n", [4, 8, 16, 32, 64, 128])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_forward_inverse_small(F, n, dtype, tiny, monkeypatch):
    # both schedules of small n: the fused one-CTA-per-plane kernels (n <= 64, default) and the
    # persistent two-pass kernels (FFST_TINY=0)
    if n > 64 and tiny == "0":
        pytest.skip("n > 64 always runs the persistent kernels")
    monkeypatch.setenv("FFST_TINY", tiny)
    batch = 3
    x, xo = images(2, batch, n, dtype)
    plan = F.Plan(n, batch, dtype)
    c = plan.forward(x.cuda())
    rec = plan.inverse(c)
    torch.cuda.synchronize()
    c = c.cpu().numpy()
    rec = rec.cpu().numpy()
    psi = O.shearlet_spectra(n)
    for b in range(batch):
        ref = O.forward(xo[b], psi=psi)
        assert plane_err(c[b], ref, np.max(np.abs(xo[b]))).max() <= TOL[dtype], (n, b)
        # inverse of the GPU cube vs the oracle's inverse of the same cube (adjoint on its input)
        ref_inv = O.inverse(c[b].astype(np.complex128), psi=psi).real
        assert plane_err(rec[b], ref_inv).max() <= TOL[dtype]
        # exactness
        assert plane_err(rec[b], xo[b]).max() <= TOL[dtype]


def test_config1_float64(F):
    # BASELINE.json configs[0]: 64x64 float64 single image, forward then inverse, 1e-10
    x, xo = images(1, 1, 64, torch.float64)
    plan = F.Plan(64, 1, torch.float64)
    c = plan.forward(x.cuda())
    rec = plan.inverse(c)
    ref = O.forward(xo[0])
    assert plane_err(c.cpu().numpy()[0], ref).max() <= 1e-10
    assert plane_err(rec.cpu().numpy()[0], xo[0]).max() <= 1e-10
    assert np.max(np.abs(rec.cpu().numpy()[0] - xo[0])) < 1e-12


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_inverse_random_cube_adjoint(F, dtype):
    # the inverse on cubes outside the range of the forward (adjoint identity)
    n, batch = 64, 2
    plan = F.Plan(n, batch, dtype)
    z = synth.random_cube((batch, plan.eta, n, n), 7)
    zt = torch.from_numpy(z).to(plan.cdtype)
    zo = zt.to(torch.complex128).numpy()
    rec = plan.inverse(zt.cuda()).cpu().numpy()
    psi = O.shearlet_spectra(n)
    for b in range(batch):
        ref = O.inverse(zo[b], psi=psi).real
        assert plane_err(rec[b], ref).max() <= TOL[dtype]
    # Re <T f, Z> = <f, T* Z>
    x, xo = images(2, batch, n, dtype)
    c = plan.forward(x.cuda()).cpu().numpy().astype(np.complex128)
    lhs = np.real(np.sum(c * np.conj(zo)))
    rhs = np.sum(xo * rec)
    assert abs(lhs - rhs) <= (1e-9 if dtype == torch.float64 else 1e-4) * abs(lhs)


def test_tiny_path_matches_persistent_and_is_deterministic(F, monkeypatch):
    # the fused small-n kernels and the persistent kernels compute the same transform (to
    # rounding); the fused inverse sums the planes in a fixed order: bitwise reproducible
    n, batch = 64, 4
    x, xo = images(2, batch, n, torch.float64)
    xd = x.cuda()
    monkeypatch.setenv("FFST_TINY", "0")
    ref_plan = F.Plan(n, batch, torch.float64)
    monkeypatch.setenv("FFST_TINY", "1")
    plan = F.Plan(n, batch, torch.float64)
    c0 = ref_plan.forward(xd)
    c1 = plan.forward(xd)
    assert float((c0 - c1).abs().max() / c0.abs().max()) <= 1e-13
    r1 = plan.inverse(c1).clone()
    assert torch.equal(r1, plan.inverse(c1))
    assert float((r1 - ref_plan.inverse(c0)).abs().max()) <= 1e-13
    assert torch.equal(plan.forward(xd[1:3]), c1[1:3])


def test_constant_image(F):
    n = 64
    plan = F.Plan(n, 1, torch.float64)
    c = plan.forward(torch.full((1, n, n), 0.7, dtype=torch.float64, device="cuda")).cpu().numpy()[0]
    assert np.max(np.abs(c[0] - 0.7)) < 1e-13
    assert np.max(np.abs(c[1:])) < 1e-13


def test_batch_subset_and_determinism(F):
    n, batch = 128, 4
    x, _ = images(2, batch, n, torch.float32)
    plan = F.Plan(n, batch, torch.float32)
    c_all = plan.forward(x.cuda()).clone()
    c_one = plan.forward(x[2:3].cuda())
    assert torch.equal(c_all[2:3], c_one)          # same arithmetic whatever the batch
    c_again = plan.forward(x.cuda())
    assert torch.equal(c_all, c_again)             # bitwise deterministic (no atomics)
    r1 = plan.inverse(c_all).clone()
    r2 = plan.inverse(c_all)
    assert torch.equal(r1, r2)


def test_determinism_config2(F):
    # at the bench's launch configuration (paired forward items, accumulator lanes, the side stream
    # of the Nyquist correction): bitwise reproducible, and each image's result independent of the
    # batch it is computed in (same arithmetic, same summation order)
    cfg = synth.config(2)
    x, _ = images(2, cfg.batch, cfg.n, torch.float32)
    xd = x.cuda()
    plan = F.Plan(cfg.n, cfg.batch, torch.float32)
    c1 = plan.forward(xd).clone()
    c2 = plan.forward(xd)
    assert torch.equal(c1, c2)
    r1 = plan.inverse(c1).clone()
    r2 = plan.inverse(c1)
    assert torch.equal(r1, r2)
    c_sub = plan.forward(xd[5:8])
    assert torch.equal(c1[5:8], c_sub)
    r_sub = plan.inverse(c1[5:8].contiguous())
    assert torch.equal(r1[5:8], r_sub)


@pytest.mark.parametrize("policy", ["lpt", "round_robin"])
def test_shards_sum_to_full(F, policy):
    # eta-sharding: each shard's cube holds its planes (ffst_shard_planes); the partial images
    # (no communicator: the caller reduces) sum to the full inverse
    n, batch, shards = 64, 2, 3
    x, xo = images(2, batch, n, torch.float64)
    full = F.Plan(n, batch, torch.float64)
    c_full = full.forward(x.cuda()).cpu()
    rec_sum = torch.zeros(batch, n, n, dtype=torch.float64)
    owned = []
    for r in range(shards):
        p = F.Plan(n, batch, torch.float64, shard_rank=r, shard_count=shards, shard_policy=policy)
        assert p.local_planes == F.shard_planes(n, shards, r, policy)
        owned += p.local_planes
        c = p.forward(x.cuda())
        assert torch.allclose(c.cpu(), c_full[:, p.local_planes], atol=1e-13, rtol=0)
        rec_sum += p.inverse(c).cpu()
    assert sorted(owned) == list(range(full.eta))
    assert np.max(np.abs(rec_sum.numpy() - xo)) < 1e-12


@pytest.mark.parametrize("n,batch,dtype", [(64, 1, torch.float64), (256, 16, torch.float32), (128, 5, torch.float32)])
def test_nccl_single_rank(F, n, batch, dtype):
    # the library's own collectives (include/ffst.h "Multi-GPU") on a one-rank NCCL communicator
    # (the one GPU of this box): image broadcast in image groups before the spectrum kernels,
    # reduce of the adjoint spectra and Nyquist corrections, final synthesis on the root --
    # bitwise the results of the plan without a communicator
    comm = F.NcclComm(1, 0, torch.cuda.current_device(), F.NcclComm.unique_id())
    try:
        x, xo = images(2, batch, n, dtype)
        xd = x.cuda()
        plain = F.Plan(n, batch, dtype)
        coll = F.Plan(n, batch, dtype, nccl_comm=comm)
        c0 = plain.forward(xd)
        c1 = coll.forward(xd)
        assert torch.equal(c0, c1)
        r0 = plain.inverse(c0)
        r1 = coll.inverse(c1, root=0)
        assert torch.equal(r0, r1)
        assert plane_err(r1.cpu().numpy(), xo).max() <= TOL[dtype]
        with pytest.raises(F.FFSTError):
            coll.inverse(c1, root=1)                       # root outside the communicator
        if batch > 1:                                      # a smaller batch (other image groups)
            assert torch.equal(coll.forward(xd[1:]), c0[1:])
            assert torch.equal(coll.inverse(c0[1:].contiguous()), plain.inverse(c0[1:].contiguous()))
        coll.close()
        plain.close()
    finally:
        comm.close()


def test_reserved_batches_do_not_allocate(F):
    # transforms never allocate device memory (include/ffst.h): a batch size is reserved first
    # (Plan.reserve -> ffst_plan_reserve), after which its first call leaves device memory as is;
    # an unreserved batch fails in the C ABI before anything is launched
    import ctypes as C
    n, batch = 128, 6
    plan = F.Plan(n, batch, torch.float32)
    x = torch.randn(3, n, n, device="cuda")
    out_c = plan.empty_coeffs(3)
    out_r = plan.empty_images(3)
    with pytest.raises(F.FFSTError):
        F.plan.check(F.lib.ffst_sheartrans_batch(plan._h, C.c_void_p(x.data_ptr()), C.c_void_p(out_c.data_ptr()),
                                                 3, None), "unreserved")
    plan.reserve(3)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    plan.forward(x, out=out_c)
    plan.inverse(out_c, out=out_r)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0
    assert float((out_r - x).abs().max() / x.abs().max()) <= 1e-4


@pytest.mark.parametrize("n", [64, 128, 45])
def test_host_variants(F, n):
    # the host-buffer entry points on the fused small-n, persistent and arbitrary-n paths
    batch = 2
    x, xo = images(2, batch, n, torch.float32)
    plan = F.Plan(n, batch, torch.float32)
    c = plan.forward_host(x.pin_memory())
    out = torch.empty(batch, n, n, dtype=torch.float32).pin_memory()
    plan.inverse_host(c, out)
    torch.cuda.synchronize()
    assert plane_err(out.numpy(), xo).max() <= 1e-4
    assert torch.equal(c, plan.forward(x.cuda()))


def test_errors(F):
    with pytest.raises(F.FFSTError):
        F.Plan(3, 1)
    with pytest.raises(F.FFSTError):
        F.Plan(4095, 1)                                  # arbitrary n: built up to 2048
    with pytest.raises(F.FFSTError):
        F.Plan(100, 1).forward_compact(torch.zeros(1, 100, 100, device="cuda"))   # compact: 2^k n only
    with pytest.raises(F.FFSTError):
        F.Plan(4096, 1, torch.float64)
    plan = F.Plan(32, 2)
    with pytest.raises(ValueError):
        plan.forward(torch.zeros(3, 32, 32, device="cuda"))


# ------------------------------------------------------------------ the benchmark configs

def _check_forward_planes(c_gpu, x64, planes, tol, n):
    f_hat = O.dft2_centred(x64)
    errs = []
    for i in planes:
        ref = O.forward_plane(x64, i + 1, f_hat=f_hat)
        errs.append(plane_err(c_gpu[i], ref, np.max(np.abs(x64))))
    return max(errs)


@pytest.mark.parametrize("env", [{}, {"FFST_RING_MB": "1", "FFST_CHUNK_PLANES": "2"}])
def test_config2_full(F, env, monkeypatch):
    # configs[1]: 256x256 float32 batch 16 — every plane of every image, and the inverse; also
    # with a tiny intermediate ring (every slot reused many times: the ring-reuse and
    # accumulation-chain dependencies of the persistent scheduler are exercised)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = synth.config(2)
    x, xo = images(2, cfg.batch, cfg.n, torch.float32)
    plan = F.Plan(cfg.n, cfg.batch, torch.float32)
    c = plan.forward(x.cuda())
    rec = plan.inverse(c).cpu().numpy()
    c = c.cpu().numpy()
    psi = O.shearlet_spectra(cfg.n)
    worst = 0.0
    for b in range(cfg.batch):
        ref = O.forward(xo[b], psi=psi)
        worst = max(worst, plane_err(c[b], ref, np.max(np.abs(xo[b]))).max())
        ref_inv = O.inverse(c[b].astype(np.complex128), psi=psi).real
        assert plane_err(rec[b], ref_inv).max() <= 1e-4
        assert plane_err(rec[b], xo[b]).max() <= 1e-4
    assert worst <= 1e-4, worst


def _kind_scale_planes(n, j0=None):
    """One plane of every (kind, j) pair, the low-pass, and the Nyquist planes of the finest
    scale (0-based flat indices): every window code path and every Nyquist-plane kind."""
    j0 = O.scales_for_size(n) if j0 is None else j0
    eta = O.num_shearlets(j0)
    first = {}
    for i in range(eta):
        kind, j, _ = O.index_to_params(j0, i + 1)
        first.setdefault((kind, j), i)
    return sorted(first.values()), eta


@pytest.mark.parametrize("cid,images_checked", [(3, (0, 63)), (4, (0, 31))])
def test_config_full_batch(F, cid, images_checked):
    # configs[2], configs[3] at their full batch (the bench launch configuration): every plane of
    # the first and last image against the oracle (forward), the full-batch inverse of the GPU
    # cube element-wise against the oracle's inverse of the same cube on those images; round trip
    # and Parseval on every image
    cfg = synth.config(cid)
    x, _ = images(cid, cfg.batch, cfg.n, torch.float32)
    plan = F.Plan(cfg.n, cfg.batch, torch.float32)
    xd = x.cuda()
    c = plan.forward(xd)
    rec = plan.inverse(c)
    err_rt = (rec - xd).abs().amax(dim=(1, 2)) / xd.abs().amax(dim=(1, 2))
    assert float(err_rt.max()) <= 1e-4
    energy_c = (c.abs() ** 2).double().sum(dim=(1, 2, 3))
    energy_f = (xd.double() ** 2).sum(dim=(1, 2))
    assert float(((energy_c - energy_f).abs() / energy_f).max()) <= 1e-4
    eta = plan.eta
    rec = rec.cpu().numpy()
    for b in images_checked:
        cb = c[b].cpu().numpy()
        x64 = x[b].double().numpy()
        ref = OP.forward_planes(x64, list(range(eta)))
        worst = max(plane_err(cb[i], ref[i], np.max(np.abs(x64))) for i in range(eta))
        assert worst <= 1e-4, (b, worst)
        ref_inv = OP.inverse(cb.astype(np.complex128), list(range(eta))).real
        assert plane_err(rec[b], ref_inv) <= 1e-4, b
    del c


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_adjoint_off_range_bench_geometry(F, cid):
    # the inverse of an ARBITRARY complex cube (outside the forward's range: general imaginary
    # parts, so the Nyquist correction's Im terms matter) at each config's full batch and launch
    # geometry (queues, ring, accumulator lanes, pass-1 item sizes): non-zero on one plane of every
    # (kind, j) pair plus finest-scale Nyquist planes of both cones, in the first and last image;
    # compared element-wise with the oracle's inverse (eq:inverseShearletTransform)
    cfg = synth.config(cid)
    n, B = cfg.n, cfg.batch
    plan = F.Plan(n, B, torch.float32)
    base, eta = _kind_scale_planes(n)
    nyq = [i for i in range(eta) if F.plane_is_nyquist(n, i)]
    sample = sorted(set(base) | {nyq[0], nyq[len(nyq) // 2], nyq[-1]})
    checked = sorted({0, B - 1})
    z = torch.zeros(B, eta, n, n, dtype=torch.complex64, device="cuda")
    zo = {}
    for b in checked:
        zb = synth.random_cube((len(sample), n, n), 1000 * cid + b).astype(np.complex64)
        z[b, sample] = torch.from_numpy(zb).cuda()
        zo[b] = zb.astype(np.complex128)
    rec = plan.inverse(z).cpu().numpy()
    for b in checked:
        ref = OP.inverse(zo[b], sample).real
        assert plane_err(rec[b], ref) <= 1e-4, b
    others = [b for b in range(B) if b not in checked]
    if others:
        assert np.max(np.abs(rec[others])) == 0.0


@pytest.mark.parametrize("n", [1024, 2048])
def test_float64_large(F, n):
    # float64 at large n (the column passes store columns straight from registers, in pairs): one
    # plane of every (kind, j) pair and Nyquist planes against the oracle at 1e-10, round trip
    x, xo = images(4, 1, n, torch.float64)
    plan = F.Plan(n, 1, torch.float64)
    xd = x.cuda()
    c = plan.forward(xd)
    rec = plan.inverse(c)
    assert float((rec - xd).abs().max() / xd.abs().max()) <= 1e-10
    base, eta = _kind_scale_planes(n)
    nyq = plan.nyquist_planes()
    planes = sorted(set(base) | {nyq[0], nyq[-1]})
    ref = OP.forward_planes(xo[0], planes)
    for i in planes:
        assert plane_err(c[0, i].cpu().numpy(), ref[i], np.max(np.abs(xo[0]))) <= 1e-10, i


def test_float32_large_two_images(F):
    # n = 2048 float32, two images (the forward intermediate in 4-row blocks, the row pass's
    # per-line tiles with LPR = 4 lines per CTA): one plane of every (kind, j) pair and the first /
    # last Nyquist planes of both images against the oracle, round trip
    n = 2048
    x, xo = images(5, 2, n, torch.float32)
    plan = F.Plan(n, 2, torch.float32)
    xd = x.cuda()
    c = plan.forward(xd)
    rec = plan.inverse(c)
    assert float((rec - xd).abs().max() / xd.abs().max()) <= 1e-4
    base, eta = _kind_scale_planes(n)
    nyq = plan.nyquist_planes()
    planes = sorted(set(base) | {nyq[0], nyq[-1]})
    for b in range(2):
        x64 = x[b].double().numpy()
        ref = OP.forward_planes(x64, planes)
        for i in planes:
            assert plane_err(c[b, i].cpu().numpy(), ref[i], np.max(np.abs(x64))) <= 1e-4, (b, i)


def test_config5_forward_planes(F):
    # configs[4]: 4096x4096 float32 single image; the forward against the oracle on one plane of
    # every (kind, j) pair and on every finest-scale Nyquist plane; round trip and Parseval
    cfg = synth.config(5)
    x, _ = images(5, 1, cfg.n, torch.float32)
    plan = F.Plan(cfg.n, 1, torch.float32)
    xd = x.cuda()
    c = plan.forward(xd)
    rec = plan.inverse(c)
    assert float((rec - xd).abs().max() / xd.abs().max()) <= 1e-4
    ec = float((c.abs() ** 2).double().sum())
    ef = float((xd.double() ** 2).sum())
    assert abs(ec - ef) / ef <= 1e-4
    base, eta = _kind_scale_planes(cfg.n)
    j0 = plan.j0
    finest_nyq = [i for i in range(eta) if O.index_to_params(j0, i + 1)[1] == j0 - 1 and F.plane_is_nyquist(cfg.n, i)]
    assert len(finest_nyq) >= 2 ** (j0 + 1) - 4
    planes = sorted(set(base) | set(finest_nyq))
    x64 = x[0].double().numpy()
    ref = OP.forward_planes(x64, planes)
    worst = 0.0
    for i in planes:
        worst = max(worst, plane_err(c[0, i].cpu().numpy(), ref[i], np.max(np.abs(x64))))
    assert worst <= 1e-4, worst


# ------------------------------------------------------------------ compact format

@pytest.mark.parametrize("n,dtype,batch", [(8, torch.float64, 2), (64, torch.float64, 3), (32, torch.float32, 3),
                                           (256, torch.float32, 16), (512, torch.float32, 4), (1024, torch.float32, 2),
                                           (4096, torch.float32, 1)])
def test_compact_format(F, n, dtype, batch):
    # the compact cube (real parts + Nyquist vectors) expands (ffst_expand_compact) to the complex
    # forward's cube, its inverse equals the complex inverse of that cube, and the round trip is
    # exact; plane by plane at large n (the cubes are 34 GB at n = 4096)
    x, xo = images(2, batch, n, dtype)
    xd = x.cuda()
    plan = F.Plan(n, batch, dtype)
    c = plan.forward(xd)
    re, gh = plan.forward_compact(xd)
    tol = 1e-5 if dtype == torch.float32 else 1e-12
    if n <= 512:
        ce = plan.expand_compact(re, gh)
        scale = c.abs().amax(dim=(2, 3), keepdim=True).clamp_min(1e-30)
        assert float(((ce - c).abs() / scale).max()) <= tol
        r_complex = plan.inverse(ce)
    else:
        r_complex = plan.inverse(c)
        ce = plan.expand_compact(re, gh, out=c)            # in place over the complex cube
        del c
    r_compact = plan.inverse_compact(re, gh)
    assert float((r_compact - r_complex).abs().max() / r_complex.abs().max()) <= tol
    assert plane_err(r_compact.cpu().numpy(), xo).max() <= TOL[dtype]
    # the expanded cube against the oracle on one image (every plane; sampled planes above 512)
    if n <= 512:
        ref = O.forward(xo[0], psi=O.shearlet_spectra(n))
        assert plane_err(ce[0].cpu().numpy(), ref, np.max(np.abs(xo[0]))).max() <= TOL[dtype]
    else:
        base, eta = _kind_scale_planes(n)
        nyq = plan.nyquist_planes()
        planes = sorted(set(base) | {nyq[0], nyq[len(nyq) // 2], nyq[-1]})
        ref = OP.forward_planes(xo[0], planes)
        for i in planes:
            assert plane_err(ce[0, i].cpu().numpy(), ref[i], np.max(np.abs(xo[0]))) <= TOL[dtype], i
    del ce, re, gh
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ smooth variant
# The oracle evaluates eq:newPsi1 as printed, sqrt(Phi^2(w/4) - Phi^2(w)), re-done in 40-digit
# arithmetic where float64 would cancel (reading A19); the kernels use the
# cancellation-free form.  Both are exact to rounding: the classic tolerances apply.
TOL_SMOOTH = TOL


@pytest.mark.parametrize("n,dtype", [(4, torch.float64), (16, torch.float64), (64, torch.float64),
                                     (256, torch.float32), (512, torch.float32)])
def test_smooth_spectra_match_oracle(F, n, dtype):
    plan = F.Plan(n, 1, dtype, variant="smooth")
    psi = plan.spectra(centred=True).cpu().double().numpy()
    ref = O.shearlet_spectra(n, variant="smooth")
    if dtype == torch.float64:
        assert np.max(np.abs(psi**2 - ref**2)) < 1e-13
        assert np.max(np.abs(psi - ref)) < 1e-13
    else:
        assert np.max(np.abs(psi - ref)) < 2e-6
    assert np.max(np.abs(np.sum(psi**2, axis=0) - 1.0)) < (1e-13 if dtype == torch.float64 else 1e-5)
    # the classic and smooth systems are different systems
    assert np.max(np.abs(psi - O.shearlet_spectra(n))) > 1e-3 or n < 16


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64, 128, 256])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_smooth_forward_inverse_small(F, n, dtype, monkeypatch):
    batch = 3
    x, xo = images(2, batch, n, dtype)
    plan = F.Plan(n, batch, dtype, variant="smooth")
    c = plan.forward(x.cuda())
    rec = plan.inverse(c)
    torch.cuda.synchronize()
    c = c.cpu().numpy()
    rec = rec.cpu().numpy()
    psi = O.shearlet_spectra(n, variant="smooth")
    for b in range(batch):
        ref = O.forward(xo[b], psi=psi)
        assert plane_err(c[b], ref, np.max(np.abs(xo[b]))).max() <= TOL_SMOOTH[dtype], (n, b)
        ref_inv = O.inverse(c[b].astype(np.complex128), psi=psi).real
        assert plane_err(rec[b], ref_inv).max() <= TOL_SMOOTH[dtype]
        assert plane_err(rec[b], xo[b]).max() <= TOL[dtype]


def test_smooth_config2_full(F):
    # configs[1] shape with the smooth system: every plane of every image, inverse, round trip
    cfg = synth.config(2)
    x, xo = images(2, cfg.batch, cfg.n, torch.float32)
    plan = F.Plan(cfg.n, cfg.batch, torch.float32, variant="smooth")
    c = plan.forward(x.cuda())
    rec = plan.inverse(c).cpu().numpy()
    c = c.cpu().numpy()
    psi = O.shearlet_spectra(cfg.n, variant="smooth")
    for b in range(cfg.batch):
        ref = O.forward(xo[b], psi=psi)
        assert plane_err(c[b], ref, np.max(np.abs(xo[b]))).max() <= 1e-4, b
        ref_inv = O.inverse(c[b].astype(np.complex128), psi=psi).real
        assert plane_err(rec[b], ref_inv).max() <= 1e-4
        assert plane_err(rec[b], xo[b]).max() <= 1e-4


def test_smooth_large_sampled(F):
    # n = 2048 float32 (multi-slot planes in HBM): sampled planes, round trip, Parseval
    n = 2048
    x, _ = images(5, 1, n, torch.float32)
    plan = F.Plan(n, 1, torch.float32, variant="smooth")
    xd = x.cuda()
    c = plan.forward(xd)
    rec = plan.inverse(c)
    assert float((rec - xd).abs().max() / xd.abs().max()) <= 1e-4
    ec = float((c.abs() ** 2).double().sum())
    ef = float((xd.double() ** 2).sum())
    assert abs(ec - ef) / ef <= 1e-4
    eta = plan.eta
    nyq = plan.nyquist_planes()
    planes = sorted({0, 1, eta // 2, eta - 1, nyq[0], nyq[len(nyq) // 2]})
    x64 = x[0].double().numpy()
    f_hat = O.dft2_centred(x64)
    for i in planes:
        ref = O.forward_plane(x64, i + 1, f_hat=f_hat, variant="smooth")
        assert plane_err(c[0, i].cpu().numpy(), ref, np.max(np.abs(x64))) <= 1e-4, i


@pytest.mark.parametrize("n,dtype,batch", [(64, torch.float64, 2), (256, torch.float32, 4)])
def test_smooth_compact_format(F, n, dtype, batch):
    x, xo = images(2, batch, n, dtype)
    xd = x.cuda()
    plan = F.Plan(n, batch, dtype, variant="smooth")
    c = plan.forward(xd)
    re, gh = plan.forward_compact(xd)
    ce = plan.expand_compact(re, gh)
    scale = c.abs().amax(dim=(2, 3), keepdim=True).clamp_min(1e-30)
    tol = 1e-5 if dtype == torch.float32 else 1e-12
    assert float(((ce - c).abs() / scale).max()) <= tol
    r_compact = plan.inverse_compact(re, gh)
    assert plane_err(r_compact.cpu().numpy(), xo).max() <= TOL[dtype]


# ------------------------------------------------------------------ user-supplied spectra

def _user_plan(F, psi, batch, dtype, centred=True, **kw):
    t = torch.from_numpy(psi).to(dtype).cuda()
    if not centred:
        t = torch.fft.ifftshift(t, dim=(-2, -1)).contiguous()
    return F.Plan(psi.shape[-1], batch, dtype, spectra=t, centred=centred, **kw), t


@pytest.mark.parametrize("n,dtype", [(16, torch.float64), (64, torch.float64), (256, torch.float32),
                                     (1024, torch.float32)])
def test_user_spectra_builtin_system(F, n, dtype):
    # the built-in spectra passed in as precomputed Psi reproduce the built-in plan
    psi = O.shearlet_spectra(n)
    batch = 3
    x, xo = images(2, batch, n, dtype)
    plan_u, _ = _user_plan(F, psi, batch, dtype)
    plan_b = F.Plan(n, batch, dtype)
    assert plan_u.eta == plan_b.eta and plan_u.variant == "user"
    cu = plan_u.forward(x.cuda())
    cb = plan_b.forward(x.cuda())
    scale = cb.abs().amax(dim=(2, 3), keepdim=True).clamp_min(1e-30)
    tol = 1e-5 if dtype == torch.float32 else 1e-12
    assert float(((cu - cb).abs() / scale).max()) <= tol
    ru = plan_u.inverse(cu)
    assert plane_err(ru.cpu().numpy(), xo).max() <= TOL[dtype]
    # export reproduces the input and the admission numbers are those of a Parseval frame
    got = plan_u.spectra(centred=True).cpu().double().numpy()
    # (exact off the Nyquist lines; sym + anti there re-rounds)
    assert np.max(np.abs(got - psi.astype(np.float32 if dtype == torch.float32 else np.float64))) <= (
        1e-7 if dtype == torch.float32 else 1e-15)
    t, a = plan_u.spectra_check()
    assert t < (1e-5 if dtype == torch.float32 else 1e-13) and a <= (1e-6 if dtype == torch.float32 else 1e-14)


@pytest.mark.parametrize("n,eta,dtype,batch,centred", [(4, 3, torch.float64, 2, True), (16, 7, torch.float64, 3, True),
                                                       (64, 13, torch.float64, 2, False), (256, 29, torch.float32, 4, True),
                                                       (512, 9, torch.float32, 2, False), (1024, 17, torch.float32, 2, True),
                                                       (4096, 5, torch.float32, 1, False)])
def test_user_spectra_random_system(F, n, eta, dtype, batch, centred):
    # a random Parseval system with pruned column bands and asymmetric Nyquist lines
    psi = synth.random_spectra(n, eta, 100 + n)
    x, xo = images(2, batch, n, dtype)
    plan, t = _user_plan(F, psi, batch, dtype, centred=centred)
    assert plan.eta == eta
    psi_o = psi.astype(np.float32).astype(np.float64) if dtype == torch.float32 else psi
    c = plan.forward(x.cuda())
    rec = plan.inverse(c).cpu().numpy()
    c = c.cpu().numpy()
    for b in range(batch):
        ref = O.forward(xo[b], psi=psi_o)
        assert plane_err(c[b], ref, np.max(np.abs(xo[b]))).max() <= TOL[dtype], b
        ref_inv = O.inverse(c[b].astype(np.complex128), psi=psi_o).real
        assert plane_err(rec[b], ref_inv).max() <= TOL[dtype]
        assert plane_err(rec[b], xo[b]).max() <= TOL[dtype]
    got = plan.spectra(centred=True).cpu().double().numpy()
    assert np.max(np.abs(got - psi_o)) <= (1e-7 if dtype == torch.float32 else 1e-15)
    tight, asym = plan.spectra_check()
    assert tight <= (1e-5 if dtype == torch.float32 else 1e-13) and asym == 0.0


def test_user_spectra_non_parseval_and_sharded(F):
    # a non-tight system runs (the check is reported, not enforced); shards sum to the full adjoint
    n, eta = 64, 11
    psi = synth.random_spectra(n, eta, 7, parseval=False)
    x, xo = images(2, 2, n, torch.float64)
    full, _ = _user_plan(F, psi, 2, torch.float64)
    tight, _ = full.spectra_check()
    assert abs(tight - O.frame_tightness(psi)) < 1e-12
    c = full.forward(x.cuda())
    ref = O.forward(xo[0], psi=psi)
    assert plane_err(c[0].cpu().numpy(), ref, np.max(np.abs(xo[0]))).max() <= 1e-10
    r_full = full.inverse(c)
    acc = torch.zeros_like(r_full)
    for rank in range(3):
        sh, _ = _user_plan(F, psi, 2, torch.float64, shard_rank=rank, shard_count=3)
        assert sh.local_planes == list(range(rank, eta, 3))
        acc += sh.inverse(c[:, sh.local_planes].contiguous())
    assert float((acc - r_full).abs().max() / r_full.abs().max()) <= 1e-12


@pytest.mark.parametrize("n,dtype", [(32, torch.float64), (64, torch.float32), (45, torch.float64)])
def test_user_spectra_asymmetric(F, n, dtype):
    # any Psi: spectra that are not point-symmetric off the Nyquist lines run on the
    # full complex path and still match the oracle's transform with the same Psi, and invert
    psi = synth.random_spectra(n, 5, 3)
    rng = np.random.default_rng(11)
    psi = psi * (1.0 + 0.3 * rng.random(psi.shape))            # breaks the point symmetry
    psi /= np.sqrt(np.sum(psi**2, axis=0, keepdims=True))       # still a Parseval system
    x, xo = images(2, 2, n, dtype)
    plan, _ = _user_plan(F, psi, 2, dtype)
    psi_o = psi.astype(np.float32).astype(np.float64) if dtype == torch.float32 else psi
    tight, asym = plan.spectra_check()
    assert asym > 1e-3 and tight <= (1e-5 if dtype == torch.float32 else 1e-13)
    c = plan.forward(x.cuda())
    rec = plan.inverse(c).cpu().numpy()
    c = c.cpu().numpy()
    for b in range(2):
        ref = O.forward(xo[b], psi=psi_o)
        assert plane_err(c[b], ref, np.max(np.abs(xo[b]))).max() <= TOL[dtype], b
        ref_inv = O.inverse(c[b].astype(np.complex128), psi=psi_o).real
        assert plane_err(rec[b], ref_inv).max() <= TOL[dtype]
        assert plane_err(rec[b], xo[b]).max() <= TOL[dtype]


def test_user_spectra_rejections(F):
    n = 32
    psi = synth.random_spectra(n, 5, 3)
    with pytest.raises(ValueError):
        F.Plan(n, 1, torch.float64, spectra=torch.zeros(5, n, n, dtype=torch.float32, device="cuda"))


def test_builtin_spectra_check(F):
    for variant in ("classic", "smooth"):
        plan = F.Plan(128, 1, torch.float64, variant=variant)
        tight, asym = plan.spectra_check()
        assert tight < 1e-13 and asym < 1e-15


# ------------------------------------------------------------------ arbitrary n

@pytest.mark.parametrize("n", [5, 33, 63, 65, 96, 100, 127, 255, 1000])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_arbitrary_n(F, n, dtype):
    # odd and non-power-of-two sizes: every plane of both images against
    # the oracle, the inverse of the GPU cube against the oracle's inverse of it, the round trip;
    # odd n has a point-symmetric grid, so its coefficients are real
    batch = 2
    x, xo = images(2, batch, n, dtype)
    plan = F.Plan(n, batch, dtype)
    assert plan.eta == O.num_shearlets(O.scales_for_size(n))
    psi_gpu = plan.spectra(centred=True).cpu().double().numpy()
    psi = O.shearlet_spectra(n)
    assert np.max(np.abs(psi_gpu - psi)) < (1e-13 if dtype == torch.float64 else 2e-6)
    c = plan.forward(x.cuda())
    rec = plan.inverse(c).cpu().numpy()
    c = c.cpu().numpy()
    for b in range(batch):
        ref = O.forward(xo[b], psi=psi)
        assert plane_err(c[b], ref, np.max(np.abs(xo[b]))).max() <= TOL[dtype], (n, b)
        ref_inv = O.inverse(c[b].astype(np.complex128), psi=psi).real
        assert plane_err(rec[b], ref_inv).max() <= TOL[dtype]
        assert plane_err(rec[b], xo[b]).max() <= TOL[dtype]
        if n % 2 == 1:
            assert np.max(np.abs(c[b].imag)) <= TOL[dtype] * np.max(np.abs(c[b]))


@pytest.mark.parametrize("n,j0", [(64, 2), (64, 4), (100, 2), (33, 3), (256, 5)])
def test_non_default_scales(F, n, j0):
    # numOfScales: any j0 up to default + 1 (reading A17); power-of-two and arbitrary n
    x, xo = images(2, 2, n, torch.float64)
    plan = F.Plan(n, 2, torch.float64, j0=j0)
    assert plan.j0 == j0 and plan.eta == O.num_shearlets(j0)
    c = plan.forward(x.cuda())
    rec = plan.inverse(c).cpu().numpy()
    c = c.cpu().numpy()
    psi = O.shearlet_spectra(n, j0)
    for b in range(2):
        assert plane_err(c[b], O.forward(xo[b], psi=psi), np.max(np.abs(xo[b]))).max() <= 1e-10
        assert plane_err(rec[b], xo[b]).max() <= 1e-10


def test_smaller_batches_all_paths(F):
    # a call with fewer images than the plan's batch (first use reserves its queue where the path
    # has one): the fused small-n path, the persistent kernels, the arbitrary-n path
    for n, path in ((32, "fused_small"), (128, "persistent"), (45, "arbitrary_n")):
        plan = F.Plan(n, 5, torch.float32)
        assert plan.path == path
        x, xo = images(2, 5, n, torch.float32)
        c_all = plan.forward(x.cuda())
        c_two = plan.forward(x[1:3].cuda())
        assert float((c_two - c_all[1:3]).abs().max()) <= 1e-6 * float(c_all.abs().max())
        r_two = plan.inverse(c_two).cpu().numpy()
        assert plane_err(r_two, xo[1:3]).max() <= 1e-4


def test_nccl_comm_must_match_the_shards(F):
    comm = F.NcclComm(1, 0, torch.cuda.current_device(), F.NcclComm.unique_id())
    try:
        with pytest.raises(F.FFSTError):
            F.Plan(64, 1, torch.float32, shard_rank=0, shard_count=2, nccl_comm=comm)
    finally:
        comm.close()


@pytest.mark.parametrize("n", [33, 100])
def test_arbitrary_n_adjoint_and_variants(F, n):
    # the adjoint on an arbitrary complex cube, the smooth system, sharding and the one-rank
    # communicator on the arbitrary-n path
    plan = F.Plan(n, 2, torch.float64)
    z = synth.random_cube((2, plan.eta, n, n), 9)
    rec = plan.inverse(torch.from_numpy(z).cuda()).cpu().numpy()
    for b in range(2):
        assert plane_err(rec[b], O.inverse(z[b]).real) <= 1e-10
    x, xo = images(2, 1, n, torch.float64)
    sm = F.Plan(n, 1, torch.float64, variant="smooth")
    cs = sm.forward(x.cuda()).cpu().numpy()[0]
    assert plane_err(cs, O.forward(xo[0], variant="smooth"), np.max(np.abs(xo[0]))).max() <= 1e-10
    c_full = plan.forward(torch.cat([x, x]).cuda())
    acc = torch.zeros(2, n, n, dtype=torch.float64, device="cuda")
    for r in range(3):
        sh = F.Plan(n, 2, torch.float64, shard_rank=r, shard_count=3)
        acc += sh.inverse(c_full[:, sh.local_planes].contiguous())
    assert float((acc[0].cpu() - torch.from_numpy(xo[0])).abs().max()) <= 1e-12
    comm = F.NcclComm(1, 0, torch.cuda.current_device(), F.NcclComm.unique_id())
    try:
        pc = F.Plan(n, 2, torch.float64, nccl_comm=comm)
        assert torch.equal(pc.forward(torch.cat([x, x]).cuda()), c_full)
        assert torch.equal(pc.inverse(c_full), plan.inverse(c_full))
        pc.close()
    finally:
        comm.close()
