"""S^(0) drawn on the device (nlsp_ctx_set_s0_draw, csrc/s0_device.cu): the
mt19937_64 words come from a tree of jump-aheads and must be bit for bit the
host generator's; the Box-Muller normals use CUDA's log / sincos and may differ
from the reference's (glibc) in their last bits, so they are compared by ulp
distance, and the whole pipeline built on them is held to the same reference
goldens and north-star tolerances as the host draw."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import check_basis_coarse_sketch, golden
from paper_2601_20174_b200 import _lib as L
from paper_2601_20174_b200 import problems

pytestmark = pytest.mark.gpu


def _host_words(seed, count):
    out = np.empty(count, dtype=np.uint64)
    L.inputs_lib().nlsp_mt19937_64_fill(seed, 0, count, L.u64ptr(out))
    return out


@pytest.mark.parametrize("count", [1, 311, 1000, (1 << 18) + 5, 3 * (1 << 18), (1 << 24) + 7])
def test_device_words_are_the_host_generator(nlsp, count):
    # one substream, a substream boundary, a full tree of 65 substreams
    ctx = nlsp.default_context()
    assert np.array_equal(ctx.mt19937_64_words(20174, count), _host_words(20174, count))


def _ulp_distance(a, b):
    ia = a.view(np.int64).copy()
    ib = b.view(np.int64).copy()
    ia[ia < 0] = np.iinfo(np.int64).min - ia[ia < 0]
    ib[ib < 0] = np.iinfo(np.int64).min - ib[ib < 0]
    return np.abs(ia - ib)


@pytest.fixture
def device_draw(nlsp):
    ctx = nlsp.default_context()
    ctx.set_s0_draw("device")
    try:
        yield ctx
    finally:
        ctx.set_s0_draw("host")


@pytest.mark.parametrize("cfg,nx,m", [("C4", 64, None), ("C5", 320, None), ("C1", 33, 7)])
def test_device_s0_is_the_reference_stream_to_the_last_bits(nlsp, device_draw, cfg, nx, m):
    """No sweeps: S^(0) itself. C5's clamped edge takes the masked scatter; C1
    at 33 x 33 with m = 7 has an odd element count (the last pair's sine is
    dropped, its second uniform still drawn)."""
    c = problems.CONFIGS[cfg].scaled(nx=nx)
    pb = problems.generate(c)
    a = pb.csr()
    mm = m or c.m
    mask = pb.mask if pb.mask.any() else None
    s = nlsp.generate_smoothed_vectors(a, mask, mm, 0, c.omega, c.s0_seed).s.numpy()
    assert device_draw.last_s0_draw() == "device"
    ref = problems.smoothed_s0(c.s0_seed, pb.n, mm, mask)
    assert s.shape == ref.shape
    if mask is not None:
        assert not s[mask.astype(bool)].any()
    ulp = _ulp_distance(s.ravel(), ref.ravel())
    frac = float((ulp > 0).mean())
    print(f"{cfg}: {s.size} normals, {frac:.2%} differ from glibc's, max {int(ulp.max())} ulp")
    assert ulp.max() <= 8 and frac < 0.5
    assert np.abs(s - ref).max() <= 1e-15 * np.abs(ref).max()


def test_host_draw_stays_the_default_and_bitwise(nlsp):
    c = problems.CONFIGS["C1"]
    pb = problems.generate(c)
    s = nlsp.generate_smoothed_vectors(pb.csr(), None, c.m, 0, c.omega, c.s0_seed).s.numpy()
    assert nlsp.default_context().last_s0_draw() == "host"
    assert np.array_equal(s, problems.smoothed_s0(c.s0_seed, pb.n, c.m, None))


@pytest.mark.parametrize("name", ["mid_C4", "mid_C5"])
def test_pipeline_on_device_drawn_vectors_matches_reference(nlsp, device_draw, name):
    """bench_single's SVD row at mid size with S^(0) drawn on the device,
    against the reference's own run: same tolerances as test_gpu_midsize.py."""
    d = golden(name)
    cfg = problems.CONFIGS[name[4:]].scaled(nx=int(d["nx"]))
    pb = problems.generate(cfg)
    a = pb.csr()
    mask = pb.mask if pb.mask.any() else None
    sv = nlsp.generate_smoothed_vectors(a, mask, cfg.m, cfg.s1, cfg.omega, cfg.s0_seed)
    assert device_draw.last_s0_draw() == "device"
    p, sig, _ = nlsp.svd_basis(sv.s, cfg.k)
    sref = np.asarray(d["sigma"])
    assert np.abs(np.asarray(sig) - sref[: len(sig)]).max() <= 1e-10 * sref[0]
    m = nlsp.TwoLevelPreconditioner(a, p, cfg.omega, cfg.nu1, cfg.nu2)
    basis, _, coarse = m._export()
    er, es, ea = check_basis_coarse_sketch(d, basis, coarse, cfg.k)
    res = nlsp.pcg(a, pb.rhs, m, cfg.delta, 10 * pb.n)
    rep = res.report
    x = np.asarray(d["x"])
    ex = np.linalg.norm(res.solution - x) / np.linalg.norm(x)
    print(f"{name} (device draw): P rows {er.max():.2e} sketch {es.max():.2e} A_c {ea:.2e} "
          f"iterations {rep.iterations} vs {int(d['iterations'])} x {ex:.2e}")
    assert rep.converged and abs(rep.iterations - int(d["iterations"])) <= 2
    assert rep.residual_history[-1] < cfg.delta and rep.true_relative_residual < 10 * cfg.delta
    assert ex <= 1e-9
