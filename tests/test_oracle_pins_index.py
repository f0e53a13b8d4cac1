"""Pins of the oracle's index work and of the parts that DARTS == vanilla alone
cannot separate (no GPU needed):

- R20 (Fig. 1): the emitter draw e = floor(N_e u)
  with weight N_e, and the emission start times tau_e -- by linearity of the
  transient integral in the emitters.
- R21 ("a time interval will be sampled", PAPER.md:373 per-frame
  dedicated paths): the per-pixel bin offset o_p, the bin of sample s and the
  per-cell sample count n_pb -- by brute-force counting, by the bins a render
  actually writes, and by the per-pixel estimator agreeing with the per-cell
  one.
- R14 (PAPER.md:301 case II): the time-checked Lambertian NEE and the cosine
  bounce at a box wall -- by a single-bounce 2-D quadrature over the wall.

Each test names the mistake it would catch.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

import dts_inputs as I


def _z(a, sa, b, sb):
    return (a - b) / np.sqrt(sa ** 2 + sb ** 2 + 1e-300)


# ---------------------------------------------------------------- floor(n u) as an integer
def test_uniform_index_is_the_exact_floor(oracle):
    """floor(n u) for the R24 uniform u = (r >> 9) 2^-23 (or_uniform, pinned by
    the Random123 known-answer vectors) equals the exact rational floor, on
    random draws and on both sides of every slice edge that was tried; an fp32
    product n * u (what the GPU did in round 1) fails here for n = 1000."""
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 7, 1000, 4096, 123457):
        rs = [int(x) for x in rng.integers(0, 2 ** 32, 3000, dtype=np.uint64)] + [0, 2 ** 32 - 1]
        for k in rng.integers(0, n, 60):
            m = -(-(int(k) << 23) // n)          # smallest m with floor(n m / 2^23) = k
            rs += [m << 9, (max(m - 1, 0) << 9) | 511]
        for r in rs:
            exact = math.floor(Fraction(n * (r >> 9), 2 ** 23))
            assert oracle.uniform_index(n, r) == exact, (n, r)
            assert exact == math.floor(n * oracle.uniform(r))   # n m < 2^53: the double product is exact
            assert 0 <= exact < n
    # the fp32 product of round 1 rounds up across slice edges
    bad = 0
    for k in range(1, 1000, 7):
        m = -(-(k << 23) // 1000) - 1
        u32 = np.float32(np.float32(m) * np.float32(2.0 ** -23))
        bad += int(np.floor(np.float32(1000.0) * u32)) != oracle.uniform_index(1000, m << 9)
    assert bad > 0


# ---------------------------------------------------------------- R21
def test_r21_pixel_offsets_are_uniform(oracle):
    """o_p = floor(B u_p) over many pixels is uniform on 0..B-1 (chi-square):
    catches an offset taken from the wrong word / scale (e.g. always 0)."""
    c = I.config(5)
    B = c["n_bins"]
    o = np.array([oracle.pixel_offset(c, c["seed"], p) for p in range(0, 60000)])
    assert o.min() >= 0 and o.max() < B
    cnt = np.bincount(o, minlength=B)
    chi2 = ((cnt - len(o) / B) ** 2 / (len(o) / B)).sum()
    assert stats.chi2.sf(chi2, B - 1) > 1e-3
    # a different seed gives different offsets (the seed keys the draw)
    o2 = np.array([oracle.pixel_offset(c, c["seed"] + 1, p) for p in range(0, 2000)])
    assert np.mean(o2 == o[:2000]) < 0.01


@pytest.mark.parametrize("B,spp", [(1, 5), (7, 3), (7, 7), (7, 23), (1000, 1024), (1000, 999), (1000, 1), (128, 192)])
def test_r21_cell_counts_by_brute_force(oracle, B, spp):
    """n_pb equals the count of samples s in [0, spp) whose bin (s + o_p) mod B
    is b, and sums to spp over the bins: catches an off-by-one in the
    remainder rule or a count that ignores the offset."""
    c = dict(I.config(5), n_bins=B)
    for p in (0, 1, 517, 1048575):
        o = oracle.pixel_offset(c, 4, p)
        brute = np.bincount([(s + o) % B for s in range(spp)], minlength=B)
        got = np.array([oracle.cell_count(c, spp, o, b) for b in range(B)])
        np.testing.assert_array_equal(got, brute)
        assert got.sum() == spp


def test_r21_render_writes_only_the_bins_of_its_samples(oracle):
    """A per-pixel render with spp = 3 writes into bins (o_p + s) mod B,
    s = 0, 1, 2, of each pixel and nowhere else (catches a decode that puts
    sample s into another bin, e.g. (s - o_p) mod B); most of those cells get
    signal."""
    c = I.as_f32(I.small(I.config(5), 5, 4, n_bins=40, t1=40.0))
    q, _ = oracle.build_table(c)
    h = oracle.render(c, q, 3, 7, sq=False)["hist"]
    allowed = np.zeros_like(h, bool)
    for py in range(4):
        for px in range(5):
            o = oracle.pixel_offset(c, 7, py * c["width"] + px)
            for s in range(3):
                allowed[py, px, (o + s) % c["n_bins"]] = True
    assert not (h[~allowed] != 0).any()
    # bins before the first arrival (t < 4) are empty whatever the offset
    early = np.zeros_like(allowed)
    early[..., :4] = True
    assert (h[allowed & ~early] > 0).mean() > 0.5   # most samples connect (a sanity check; ~2/3 do)


@pytest.mark.parametrize("case", ["cfg1_detector", "cfg5_box"])
def test_r21_pixel_mode_equals_cell_mode(oracle, case):
    """The per-pixel estimator (each sample in one bin, the cell's mean over its
    n_pb samples) and the per-cell estimator (spp samples per cell) estimate the
    same H[p, b]: catches a wrong n_pb weight (cells holding one or two samples
    each, so a weight error is a factor 2) or a wrong bin decode.  Means and SEs
    over independent seeds of the per-pixel render."""
    if case == "cfg1_detector":
        c = I.as_f32(I.config(1, spp_mode="pixel", parity_r_excl=0.3, parity_s_excess=0.05))
        spp_pix, seeds, spp_cell = 192, 3000, 20000         # 128 bins: 64 cells get 2 samples, 64 get 1
    else:
        c = I.as_f32(I.small(I.config(5, parity_s_excess=0.05), 2, 2, n_bins=8, t1=16.0))
        spp_pix, seeds, spp_cell = 12, 1200, 3000          # 8 bins: 4 cells get 2 samples, 4 get 1
    q, _ = oracle.build_table(c)
    runs = np.array([oracle.render(c, q, spp_pix, 1000 + s, sq=False, nthreads=2)["hist"] for s in range(seeds)])
    hp, sp = runs.mean(0), runs.std(0, ddof=1) / math.sqrt(seeds)
    cc = dict(c, spp_mode="cell")
    r = oracle.render(cc, q, spp_cell, 77)
    hc = r["hist"]
    sc = np.sqrt(np.maximum(r["hist_sq"] - hc ** 2, 0) / (spp_cell - 1))
    m = (hp > 0) | (hc > 0)
    z = _z(hp, sp, hc, sc)[m]
    print(f"{case}: cells {m.sum()} within-3SE {np.mean(np.abs(z) < 3):.3f} mean z {z.mean():+.3f}")
    assert m.sum() >= 6
    assert (np.abs(z) >= 3).sum() <= max(1, int(0.01 * m.sum())), z
    assert hp[m].sum() == pytest.approx(hc[m].sum(), rel=0.1)


# ---------------------------------------------------------------- R20
def test_r20_emitters_add_linearly(oracle):
    """Light transport is linear in the sources: the two-emitter render of
    config 4 (tau = 0 and 1.5) equals the sum of the two single-emitter renders,
    each with its own start time.  Catches a dropped N_e weight (the sum halves),
    a biased emitter draw, or tau_e of the wrong emitter."""
    c = I.as_f32(I.small(I.config(4, parity_r_excl=0.3, parity_s_excess=0.05), 3, 3))
    n = 40000

    def run(cc, seed):
        q, _ = oracle.build_table(cc)
        r = oracle.render(cc, q, n, seed)
        h = r["hist"]
        return h, np.sqrt(np.maximum(r["hist_sq"] - h ** 2, 0) / (n - 1))

    h2, s2 = run(c, 31)
    h0, s0 = run(dict(c, emitters=[c["emitters"][0]]), 32)
    h1, s1 = run(dict(c, emitters=[c["emitters"][1]]), 33)
    assert h0.sum() > 0 and h1.sum() > 0
    # both emitters matter in this gate: neither is negligible against the other
    assert 0.1 < h0.sum() / h1.sum() < 10
    hs, ss = h0 + h1, np.sqrt(s0 ** 2 + s1 ** 2)
    m = (h2 > 0) | (hs > 0)
    z = _z(h2, s2, hs, ss)[m]
    print(f"R20 linearity: cells {m.sum()} z {np.round(z, 2)}")
    assert (np.abs(z) >= 3).sum() <= 1
    tot = (h2.sum() - hs.sum()) / math.sqrt((s2 ** 2).sum() + (ss ** 2).sum())
    assert abs(tot) < 3


# ---------------------------------------------------------------- R14 box walls
def _wall_config(strategy):
    """A box [-2, 2]^2 x [-1, 3] whose -z face (z = -1) is a Lambertian wall of
    albedo 0.8, every other face open, in an almost non-scattering medium
    (sigma_s = 1e-4); a pulse emitter and a fluence detector 1 above the wall."""
    return I.as_f32(I.config(1, sigma_s=1e-4, sigma_a=0.05, medium="box", bmin=(-2.0, -2.0, -1.0),
                             bmax=(2.0, 2.0, 3.0), wall_mask=1 << 4, wall_albedo=(0.0, 0.0, 0.0, 0.0, 0.8, 0.0),
                             emitters=[((0.5, 0.0, 0.0), 0.0, 1.0)], cam_pos=(-0.5, 0.0, 0.0), det_radius=0.02,
                             t0=2.0, t1=6.0, n_bins=40, strategy=strategy, name="box_wall_single_bounce"))


def _wall_single_bounce(c, edges, N=1500):
    """Bin-integrated fluence at the detector centre from one Lambertian bounce
    off the wall: sum over wall points y of P/(4 pi) cos_i e^{-st r1} / r1^2
    (rho / pi) cos_o e^{-st r2} / r2^2 dA, binned by t = r1 + r2 (midpoint
    rule on an N x N grid of the face)."""
    (xe, te, P), = c["emitters"]
    xe, xd = np.asarray(xe), np.asarray(c["cam_pos"])
    st = c["sigma_s"] + c["sigma_a"]
    rho = c["wall_albedo"][4]
    zw = c["bmin"][2]
    (x0, y0), (x1, y1) = c["bmin"][:2], c["bmax"][:2]
    hx, hy = (x1 - x0) / N, (y1 - y0) / N
    X, Y = np.meshgrid(x0 + hx * (np.arange(N) + 0.5), y0 + hy * (np.arange(N) + 0.5), indexing="ij")
    y = np.stack([X, Y, np.full_like(X, zw)], -1)
    v1, v2 = xe - y, xd - y
    r1, r2 = np.linalg.norm(v1, axis=-1), np.linalg.norm(v2, axis=-1)
    ci, co = v1[..., 2] / r1, v2[..., 2] / r2
    val = P / (4 * math.pi) * ci * np.exp(-st * r1) / r1 ** 2 * (rho / math.pi) * co * np.exp(-st * r2) / r2 ** 2 * hx * hy
    return np.histogram((te + r1 + r2).ravel(), bins=edges, weights=val.ravel())[0]


@pytest.mark.parametrize("strategy", ["darts", "vanilla"])
def test_box_wall_single_bounce_quadrature(oracle, strategy):
    """The whole estimator with one box wall (the R14 wall vertex: time-checked
    direct NEE with albedo / pi and the cosine at the wall, cosine-hemisphere
    bounce; vanilla: the same wall NEE binned by arrival time) against a 2-D
    quadrature of the single bounce over the wall.  Catches a wrong wall
    constant (albedo, 1/pi), a missing cosine, a wrong face or plane, or a
    time check that drops or double-counts wall-last paths.  Bins to 3 SE + 1 %,
    the sum to 2 %."""
    c = _wall_config(strategy)
    edges = np.linspace(c["t0"], c["t1"], c["n_bins"] + 1)
    ref = _wall_single_bounce(c, edges)
    q = oracle.build_table(c)[0] if strategy == "darts" else None
    spp = 1000 if strategy == "darts" else 100000
    runs = np.array([oracle.render(c, q, spp, seed, sq=False)["hist"][0, 0] for seed in range(16)])
    m, se = runs.mean(0), runs.std(0, ddof=1) / 4.0
    ok = np.abs(m - ref) <= 3 * se + 0.01 * ref + 3e-4 * ref.max()
    print(f"wall/{strategy}: sum {m.sum():.5e} quadrature {ref.sum():.5e}; bins ok {ok.mean():.3f}")
    assert ref.sum() > 0 and (ref > 0).sum() >= 20
    assert ok.mean() >= 0.95, np.c_[m, ref, se]
    assert m.sum() == pytest.approx(ref.sum(), rel=0.02)


# ---------------------------------------------------------------- config 5: DARTS == vanilla at a mid window
def test_cfg5_darts_equals_vanilla_mid_window(oracle):
    """PAPER.md:340 ("verified to converge to the same results") at config 5's
    mid window t in [40, 50): DARTS (RIS distance, EDA + HG in SPLIT mode,
    elliptical connections) and the vanilla estimator on a 2 x 2-pixel crop,
    5 bins of 2 time units.  Per-path contributions are heavy-tailed there (a
    cell's effective sample size n_eff = (sum x)^2 / sum x^2 is ~2 per 2000
    DARTS paths), so the comparison pools: the window total and each bin summed
    over the 4 pixels, at 20 000 DARTS paths per cell and 200 000 vanilla paths
    per pixel, each within 3 SE, with n_eff reported."""
    c = I.small(I.config(5, parity_s_excess=0.05, spp_mode="cell"), 2, 2, n_bins=5, t1=50.0)
    c["t0"] = 40.0
    c = I.as_f32(c)
    q, _ = oracle.build_table(c)
    nd, nv = 20000, 200000
    d = oracle.render(c, q, nd, 51)
    v = oracle.render(dict(c, strategy="vanilla"), None, nv, 52)
    # per-cell variances of the cell means, pooled by summation (independent cells)
    vd = np.maximum(d["hist_sq"] - d["hist"] ** 2, 0) / (nd - 1)
    vv = np.maximum(v["hist_sq"] - v["hist"] ** 2, 0) / (nv - 1)
    hd, hv = d["hist"].sum(axis=(0, 1)), v["hist"].sum(axis=(0, 1))
    sd, sv = vd.sum(axis=(0, 1)), vv.sum(axis=(0, 1))
    z_bins = (hd - hv) / np.sqrt(sd + sv)
    z_tot = (hd.sum() - hv.sum()) / math.sqrt(sd.sum() + sv.sum())
    neff_d = float(np.mean(nd * d["hist"] ** 2 / np.maximum(d["hist_sq"], 1e-300)))
    neff_v = float(np.mean(nv * v["hist"] ** 2 / np.maximum(v["hist_sq"], 1e-300)))
    print(f"cfg5 [40,50): DARTS {hd.sum():.4e} vanilla {hv.sum():.4e}, z total {z_tot:+.2f}, z bins {np.round(z_bins, 2)}; "
          f"mean n_eff per cell DARTS {neff_d:.1f} vanilla {neff_v:.1f}")
    assert hd.sum() > 0 and hv.sum() > 0
    assert abs(z_tot) < 3
    assert (np.abs(z_bins) < 3).all()
