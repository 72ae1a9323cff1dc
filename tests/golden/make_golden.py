"""Generate golden vectors by running the REFERENCE itself.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

It imports ``pgtrace`` from /root/reference/pkg/src, feeds it the seeded
synthetic inputs of ``paper_2112_09728_b200.synth`` (float32, upcast to
float64 as the reference does) and stores inputs + reference outputs as
compressed .npz files next to this script.  The GPU box never runs this;
tests load the committed .npz files.

Files:
  seq_64x48.npz    6-frame sequence, spp=2: reproject -> depth-0 sampling
                   (after 3 NEE draws) -> training_pass, chained through the
                   reference's own Gamma.
  trained_48x40.npz one frame from a randomly "pre-trained" Gamma (k in
                   [0, 90], correlated lobes, resets), same three stages.
  kat.npz          PCG32 vectors, sgmap round trips, lobe_from_stats on 4000
                   random stats, m_step_update batches, box_muller.
"""

import os
import sys
from types import SimpleNamespace

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

from pgtrace import guide_buffers as gb  # noqa: E402
from pgtrace import mixture, ptrace, rng, sgmap  # noqa: E402

from paper_2112_09728_b200 import synth  # noqa: E402

GB_FIELDS = ("valid", "pos", "normal", "depth", "mat", "kind", "albedo", "roughness", "front", "view",
             "motion", "has_history")
VPL_FIELDS = ("valid", "y", "radiance", "strategy")


def to_ref_gbuf(d):
    f = {}
    for k in GB_FIELDS:
        a = d[k].cpu().numpy()
        f[k] = a.astype(np.float64) if a.dtype == np.float32 else a
    return ptrace.GBuffer(width=d["width"], height=d["height"], cam_origin=np.array(d["cam_origin"], dtype=np.float64),
                          **f)


def to_ref_vpl(v):
    return ptrace.VplBuffer(valid=v["valid"].cpu().numpy(), y=v["y"].cpu().numpy().astype(np.float64),
                            radiance=v["radiance"].cpu().numpy().astype(np.float64),
                            strategy=v["strategy"].cpu().numpy())


def ref_scene(seed):
    kind, rough, alb = synth._materials(seed, "cpu")
    return SimpleNamespace(mat_kind=kind.numpy().astype(np.int64), mat_rough=rough.numpy().astype(np.float64),
                           mat_albedo=alb.numpy().astype(np.float64))


def ref_sample(scene, g, stats_f32, seed, frame, spp, nee_draws=3, rough_min=0.05):
    """Depth-0 lanes exactly as pg/ptrace.py:_render_chunk/_trace_lanes issue them."""
    h, w = g.height, g.width
    p = h * w
    stats = stats_f32.reshape(-1, 8).astype(np.float64)
    lobe = mixture.lobe_from_stats(stats)
    valid = g.valid.reshape(-1)
    kind = g.kind.reshape(-1)
    rough = g.roughness.reshape(-1)
    guided = valid & ((kind == 0) | (rough >= rough_min)) & (stats[:, mixture.EPOCH] >= 1.0)
    pix = np.nonzero(valid)[0]
    out = dict(wi=np.zeros((p, spp, 3)), pdf=np.zeros((p, spp)), strategy=np.zeros((p, spp), np.uint8),
               valid=np.zeros((p, spp), bool), state=np.zeros((p, spp), np.uint64))
    lob = mixture.GaussianLobe(lobe.mu[pix], lobe.cov[pix], lobe.chol[pix], lobe.trunc_z[pix])
    for s in range(spp):
        streams = rng.make_streams(seed, frame, pix.astype(np.int64) * spp + s)
        for _ in range(nee_draws):
            rng.next_f64(streams)
        mat = np.maximum(g.mat.reshape(-1)[pix], 0)
        wi, pdf, st, ok = ptrace._sample_first_bounce(
            scene, np.arange(pix.size), g.pos.reshape(-1, 3)[pix], g.normal.reshape(-1, 3)[pix], mat,
            g.view.reshape(-1, 3)[pix], stats[pix], lob, guided[pix], streams)
        out["wi"][pix, s] = wi
        out["pdf"][pix, s] = pdf
        out["strategy"][pix, s] = st
        out["valid"][pix, s] = ok
        out["state"][pix, s] = streams
    return out


def pack_inputs(prefix, gbd, vd):
    z = {}
    for k in GB_FIELDS:
        z[f"{prefix}gb_{k}"] = gbd[k].cpu().numpy()
    z[f"{prefix}gb_cam_origin"] = np.array(gbd["cam_origin"], dtype=np.float64)
    for k in VPL_FIELDS:
        z[f"{prefix}vpl_{k}"] = vd[k].cpu().numpy()
    return z


def make_seq(path, w=64, h=48, frames=6, seed=3, spp=2):
    scene = ref_scene(seed)
    z = dict(width=w, height=h, frames=frames, seed=seed, spp=spp)
    gamma = gb.GuidingBuffer.create(w, h)
    gprev = None
    for f, (gbd, vd) in enumerate(synth.sequence(w, h, frames, seed=seed)):
        g = to_ref_gbuf(gbd)
        v = to_ref_vpl(vd)
        z.update(pack_inputs(f"f{f}_", gbd, vd))
        z[f"f{f}_gamma_in"] = gamma.stats.copy()
        if gprev is not None:
            gamma = gb.reproject(gamma, gprev, g, gb.ReprojectionPolicy())
        z[f"f{f}_gamma_reproj"] = gamma.stats.copy()
        smp = ref_sample(scene, g, gamma.stats, seed, f, spp)
        for k, a in smp.items():
            z[f"f{f}_smp_{k}"] = a
        gamma = gb.training_pass(gamma, v, g, k_max=64, seed=seed, frame_index=f)
        z[f"f{f}_gamma_trained"] = gamma.stats.copy()
        gprev = g
    np.savez_compressed(path, **z)


def random_trained_stats(h, w, seed):
    """Plausible trained Gamma: lobes inside the square, some tight, some
    strongly correlated, a few indefinite (-> reset), k in [0, 90]."""
    r = np.random.default_rng(seed)
    p = h * w
    mu = r.uniform(0.05, 0.95, (p, 2))
    sd = 10 ** r.uniform(-1.9, -0.4, (p, 2))
    rho = r.uniform(-0.97, 0.97, p)
    cxy = rho * sd[:, 0] * sd[:, 1]
    st = np.zeros((p, 8))
    st[:, 0:2] = mu
    st[:, 2] = sd[:, 0] ** 2 + mu[:, 0] ** 2 - 1e-4 * r.uniform(0, 1, p)
    st[:, 3] = sd[:, 1] ** 2 + mu[:, 1] ** 2 - 1e-4 * r.uniform(0, 1, p)
    st[:, 4] = cxy + mu[:, 0] * mu[:, 1]
    bad = r.uniform(0, 1, p) < 0.1
    st[bad, 4] += r.choice([-1, 1], bad.sum()) * 0.3
    st[:, 5] = r.exponential(1.0, p)
    st[:, 6] = r.uniform(0.05, 0.95, p)
    st[:, 7] = r.integers(0, 91, p)
    zero = r.uniform(0, 1, p) < 0.1
    st[zero, 7] = 0
    return st.reshape(h, w, 8).astype(np.float32)


def make_trained(path, w=48, h=40, seed=5, spp=3, frame=7):
    scene = ref_scene(seed)
    z = dict(width=w, height=h, seed=seed, spp=spp, frame=frame)
    seq = list(synth.sequence(w, h, 2, seed=seed, first_frame=frame - 1))
    (gbp, _), (gbd, vd) = seq
    z.update(pack_inputs("p_", gbp, vd))
    z.update(pack_inputs("c_", gbd, vd))
    gprev, g, v = to_ref_gbuf(gbp), to_ref_gbuf(gbd), to_ref_vpl(vd)
    st = random_trained_stats(h, w, seed)
    z["gamma_in"] = st
    gamma = gb.reproject(gb.GuidingBuffer(w, h, st), gprev, g, gb.ReprojectionPolicy())
    z["gamma_reproj"] = gamma.stats.copy()
    # sampling and training straight from the pre-trained Gamma (no reprojection)
    smp = ref_sample(scene, g, st, seed, frame, spp)
    for k, a in smp.items():
        z[f"smp_{k}"] = a
    z["gamma_trained"] = gb.training_pass(gb.GuidingBuffer(w, h, st), v, g, k_max=64, seed=seed,
                                          frame_index=frame).stats.copy()
    z["gamma_trained_r7"] = gb.training_pass(gb.GuidingBuffer(w, h, st), v, g, k_max=32, seed=seed,
                                             frame_index=frame, neighbor_radius=7.3).stats.copy()
    np.savez_compressed(path, **z)


def make_kat(path):
    z = {}
    s = rng.make_streams(0, 0, np.arange(4))
    z["pcg_0_0_a"] = rng.next_u32(s)
    z["pcg_0_0_b"] = rng.next_u32(s)
    s = rng.make_streams(3, 1, np.array([0, 1]), stream_id=1)
    z["pcg_3_1_s1"] = rng.next_u32(s)
    s = rng.make_streams(123456789, 77, np.arange(1000, 1064, dtype=np.int64) * 7, stream_id=0)
    z["pcg_big_state0"] = s.copy()
    z["pcg_big"] = np.stack([rng.next_u32(s) for _ in range(40)])
    r = np.random.default_rng(11)
    sqp = r.uniform(0, 1, (5000, 2))
    sqp[:8] = [[0.5, 0.5], [1, 0.5], [0, 0], [1, 1], [0.5, 1], [0.25, 0.75], [0.5, 0.0], [0.0, 0.5]]
    z["sg_sq"] = sqp
    z["sg_dir"] = sgmap.square_to_hemisphere(sqp)
    z["sg_back"] = sgmap.hemisphere_to_square(z["sg_dir"])
    nr = r.normal(size=(500, 3))
    nr /= np.linalg.norm(nr, axis=-1, keepdims=True)
    nr[:3] = [[0, 0, 1], [0, 0, -1], [1, 0, 0]]
    t, b = sgmap.build_tangent_frame(nr)
    z["onb_n"], z["onb_t"], z["onb_b"] = nr, t, b
    # lobes: random moments incl. tight, correlated, indefinite, out-of-square means
    p = 4000
    mu = r.uniform(-0.2, 1.2, (p, 2))
    sd = 10 ** r.uniform(-2.2, 0.2, (p, 2))
    rho = r.uniform(-0.999, 0.999, p)
    st = np.zeros((p, 8), np.float32)
    st[:, 0:2] = mu
    st[:, 2] = sd[:, 0] ** 2 + mu[:, 0] ** 2 - 1e-4
    st[:, 3] = sd[:, 1] ** 2 + mu[:, 1] ** 2 - 1e-4
    st[:, 4] = rho * sd[:, 0] * sd[:, 1] + mu[:, 0] * mu[:, 1]
    st[::7, 4] += 0.5
    st[::11] = mixture.init_stats((1,)).astype(np.float32)
    st[::13, 4] = st[::13, 0] * st[::13, 1]
    st[:, 6] = r.uniform(0.05, 0.95, p)
    z["lobe_stats"] = st
    lob = mixture.lobe_from_stats(st.astype(np.float64))
    z["lobe_mu"], z["lobe_cov"], z["lobe_chol"], z["lobe_z"] = lob.mu, lob.cov, lob.chol, lob.trunc_z
    qp = r.uniform(0, 1, (p, 2))
    z["lobe_qp"] = qp
    z["lobe_pdf"] = mixture.gaussian_pdf_square(lob, qp)
    # m-step batches
    n = 300
    mst = st[:n].astype(np.float64)
    mst[:, 7] = r.integers(0, 100, n)
    sq = r.uniform(0, 1, (n, 20, 2))
    wgt = r.exponential(1, (n, 20))
    wgt[::5, :] = 0.0
    wgt[1::9, 3] = np.nan
    wgt[2::9, 4] = -1.0
    resp = r.uniform(0, 1, (n, 20))
    resp[3::17] = 0.0
    val = r.uniform(0, 1, (n, 20)) < 0.8
    z["ms_stats"], z["ms_sq"], z["ms_w"], z["ms_r"], z["ms_valid"] = mst, sq, wgt, resp, val
    z["ms_out"] = mixture.m_step_update(mst, sq, wgt, resp, valid=val, k_max=64)
    z["nc_k"] = np.arange(0, 100)
    z["nc_n"] = mixture.neighbor_count(z["nc_k"], 64)
    u = r.uniform(0, 1, (2, 1000))
    u[0, :3] = [0.0, 0.5, 1.0]
    z["bm_u"] = u
    z["bm_out"] = np.stack(mixture.box_muller(u[0], u[1]))
    np.savez_compressed(path, **z)


if __name__ == "__main__":
    torch.set_num_threads(4)
    make_kat(os.path.join(HERE, "kat.npz"))
    make_seq(os.path.join(HERE, "seq_64x48.npz"))
    make_trained(os.path.join(HERE, "trained_48x40.npz"))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
