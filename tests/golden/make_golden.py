"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``splatlift`` from /root/reference/pkg/src, runs the reference's
own projection (scene.py:252-312), binning (rasterizer.py:72-100),
accumulation (contributions.py:90-160), assignment (solver.py:111-172) and
novel-view rendering (rasterizer.py:133-234, maskrender.py:45-95) on seeded
inputs, and writes small ``.npz`` files next to this script.  Nothing
at test time reads /root/reference; the GPU box only sees these files.

Inputs of reference-generated fixtures are stored verbatim.  Inputs of the
larger synthetic workloads come from ``paper_2409_08270_b200.synth`` (seeded
numpy) and are stored as a sha256 digest plus the generator arguments.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import splatlift as ref  # noqa: E402
from splatlift import contributions as ref_contrib  # noqa: E402
from splatlift import scene as ref_scene  # noqa: E402
from splatlift import synth as ref_synth  # noqa: E402

from paper_2409_08270_b200 import synth as my_synth  # noqa: E402


def cam_row(v):
    return np.concatenate([[v.width, v.height, v.fx, v.fy, v.cx, v.cy, v.near_clip],
                           np.ravel(v.world_to_camera)]).astype(np.float64)


def frontal_view(width=16, height=16, focal=24.0, near_clip=0.01, view_id=0):
    # reference tests/conftest.py:12-25
    return ref.CameraView(view_id=view_id, width=width, height=height, fx=focal, fy=focal,
                          cx=width / 2.0 + 0.5, cy=height / 2.0 + 0.5,
                          world_to_camera=np.eye(4), near_clip=near_clip)


def random_scene(rng, n, box=1.2, depth_span=(2.5, 6.0)):
    # reference tests/conftest.py:39-52
    means = np.stack([rng.uniform(-box, box, n), rng.uniform(-box, box, n),
                      rng.uniform(*depth_span, n)], axis=1)
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    scales = rng.uniform(0.05, 0.35, size=(n, 3))
    opac = rng.uniform(0.1, 0.95, size=n)
    return ref.GaussianScene(means=means, rotations=quats, scales=scales, opacities=opac)


def scene_arrays(scene):
    return dict(means=scene.means, quats=scene.rotations, scales=scene.scales,
                opac=scene.opacities)


# ---------------------------------------------------------------- projection
def gen_projection():
    cases = {}
    rng = np.random.default_rng(20240811)
    s1 = random_scene(rng, 300)
    views = [frontal_view(48, 48, 60.0), ref_synth.ring_view(0, 1.1, 4.0, 64, 64, 70.0, 0.8),
             frontal_view(37, 23, 30.0, near_clip=3.0)]
    # cull corner cases: behind, exactly at near clip, offscreen, on axis
    s2 = ref.GaussianScene(
        means=[[0, 0, 2.0], [0, 0, -3.0], [40.0, 0, 2.0], [0, 0, 0.5], [0, 0, 0.0],
               [-50, 3, 2.0], [0.3, -0.2, 1.5]],
        rotations=[[1, 0, 0, 0]] * 7, scales=[[0.05, 0.05, 0.05]] * 6 + [[0.4, 0.01, 0.2]],
        opacities=[0.5] * 7)
    k = 0
    for scene in (s1, s2):
        for v in views + [frontal_view(16, 16, 24.0, near_clip=0.5)]:
            alive, mean2d, inv, z, radius, st = ref_scene._project_arrays(
                scene.means, scene.rotations, scene.scales, v)
            cases[f"c{k}"] = dict(
                **{f"in_{a}": b for a, b in scene_arrays(scene).items()}, cam=cam_row(v),
                alive=alive, mean2d=mean2d, conic=inv, depth=z, radius=radius,
                stats=np.array([st.n_input, st.n_emitted, st.n_behind, st.n_degenerate,
                                st.n_offscreen], np.int64))
            k += 1
    return cases


# ------------------------------------------------------------------- binning
def gen_binning():
    cases = {}
    rng = np.random.default_rng(7)
    scenes = [random_scene(rng, 400)]
    # heavy exact depth ties (frontal identity pose: camera z == world z)
    n = 600
    means = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n),
                      rng.choice([3.0, 3.5, 4.0], size=n)], axis=1)
    q = rng.normal(size=(n, 4))
    scenes.append(ref.GaussianScene(means=means, rotations=q,
                                    scales=rng.uniform(0.02, 0.3, (n, 3)),
                                    opacities=rng.uniform(0.1, 0.9, n)))
    views = [frontal_view(48, 48, 60.0), frontal_view(100, 37, 50.0)]
    k = 0
    for scene in scenes:
        for v in views:
            splats, _ = ref.project_scene(scene, v)
            b = ref.bin_gaussians_to_tiles(splats, v)
            offs = np.zeros(len(b.tile_lists) + 1, np.int64)
            offs[1:] = np.cumsum([len(x) for x in b.tile_lists])
            items = (np.concatenate([b.indices[x] for x in b.tile_lists])
                     if offs[-1] else np.zeros(0, np.int64))
            cases[f"c{k}"] = dict(**{f"in_{a}": c for a, c in scene_arrays(scene).items()},
                                  cam=cam_row(v), offsets=offs, items=items.astype(np.int64),
                                  tiles=np.array([b.tiles_x, b.tiles_y]))
            k += 1
    # tile_range corner cases (rasterizer.py:106-113), incl. the empty range
    tr = [(19.0, 8.0, 3, 1, 1), (-5.0, -5.0, 2, 4, 4), (63.9, 0.1, 1, 4, 4), (32.0, 16.0, 16, 4, 4),
          (1000.0, 5.0, 3, 4, 4), (8.0, 8.0, 0, 1, 1), (15.99, 16.0, 0, 2, 2)]
    cases["tile_range"] = dict(args=np.array(tr, np.float64),
                               out=np.array([ref.rasterizer.tile_range(*t) for t in tr], np.int64))
    return cases


# -------------------------------------------------------------- accumulation
def accumulate_case(scene, pairs, E, blend, store_inputs=True):
    t0 = time.perf_counter()
    A = ref.accumulate_contributions(scene, pairs, E, blend).values
    total = np.zeros((E, len(scene)))
    for v, m in pairs:
        total += ref_contrib._accumulate_view(scene, v, m, E, blend)
    dt = time.perf_counter() - t0
    assert np.array_equal(total.astype(np.float32), A)
    out = dict(A=A, A64=total, E=np.int64(E),
               floors=np.array([blend.alpha_floor, blend.transmittance_floor]))
    if store_inputs:
        out.update({f"in_{a}": c for a, c in scene_arrays(scene).items()})
        out["cams"] = np.stack([cam_row(v) for v, _ in pairs])
        out["masks"] = np.stack([m.labels for _, m in pairs])
    print(f"  accumulate N={len(scene)} V={len(pairs)} E={E}: {dt:.1f}s", flush=True)
    return out


def gen_accumulate():
    D, X = ref.DEFAULT_BLEND, ref.EXACT_BLEND
    cases = {}
    # test_contributions.py:26-36 single-Gaussian known answer
    v = frontal_view()
    s = ref.GaussianScene.from_gaussians([ref.Gaussian(center=(0, 0, 2.0), rotation=(1, 0, 0, 0),
                                                       scale=(0.15,) * 3, opacity=0.8)])
    full = ref.LabelMask(0, np.ones((16, 16), np.uint16))
    cases["kat_single_default"] = accumulate_case(s, [(v, full)], 2, D)
    cases["kat_single_exact"] = accumulate_case(s, [(v, full)], 2, X)
    # culled column (test_contributions.py:97-105)
    s = ref.GaussianScene(means=[[0, 0, 2.0], [0, 0, -5.0]], rotations=[[1, 0, 0, 0]] * 2,
                          scales=[[0.1] * 3] * 2, opacities=[0.5, 0.5])
    cases["culled"] = accumulate_case(s, [(v, full)], 2, D)
    # make_random fixtures used by the reference suite
    for seed, n, nv, w, h, e, blend, tag in [
            (11, 14, 2, 16, 16, 3, D, "d"), (5, 12, 4, 16, 16, 2, D, "d"),
            (9, 20, 3, 16, 16, 2, D, "d"), (3, 8, 2, 12, 12, 2, X, "x"),
            (100, 10, 2, 12, 12, 2, X, "x"), (501, 20, 2, 16, 16, 4, D, "d"),
            (900, 40, 2, 24, 24, 2, D, "d"), (31, 15, 3, 16, 16, 2, D, "d")]:
        fx = ref_synth.make_random(seed=seed, n_gaussians=n, n_views=nv, width=w, height=h,
                                   num_objects=e)
        cases[f"random_{seed}_{tag}"] = accumulate_case(fx.scene, fx.training_views(), e, blend)
    # denser frontal scenes with random labels, both blends
    rng = np.random.default_rng(20240811)
    for i, blend in enumerate((D, X)):
        sc = random_scene(rng, 60)
        vv = frontal_view(40, 24, 40.0)
        lab = rng.integers(0, 3, size=(24, 40), dtype=np.uint16)
        cases[f"frontal_{i}"] = accumulate_case(sc, [(vv, ref.LabelMask(0, lab))], 3, blend)
    # C1: make_two_cluster(seed=0, 10k, 8 views 128^2), all 8 GT masks
    fx = ref_synth.make_two_cluster(seed=0, n_gaussians=10_000, n_views=8, width=128,
                                    height=128, n_mask_views=8)
    pairs = [(vw, fx.masks[vw.view_id]) for vw in fx.views]
    cases["C1_default"] = accumulate_case(fx.scene, pairs, 2, D)
    c1x = accumulate_case(fx.scene, pairs[:2], 2, X, store_inputs=False)
    cases["C1_exact_2views"] = c1x
    # C1 with 20% label noise (C5 at oracle scale)
    nrng = np.random.default_rng(55)
    noisy = []
    for vw, m in pairs:
        lab = m.labels.copy()
        flip = nrng.random(lab.shape) < 0.2
        lab[flip] = nrng.integers(0, 2, size=int(flip.sum()), dtype=np.uint16)
        noisy.append((vw, ref.LabelMask(vw.view_id, lab)))
    c = accumulate_case(fx.scene, noisy, 2, D, store_inputs=False)
    c["masks"] = np.stack([m.labels for _, m in noisy])
    cases["C1_noisy"] = c
    # C2/C3-geometry synthetic workloads (inputs regenerated from seed; digest pinned)
    for name, kw in [("synth_coherent", dict(seed=7, n_gaussians=20_000, n_views=2, width=256,
                                              height=192, num_objects=8)),
                     ("synth_iid", dict(seed=8, n_gaussians=20_000, n_views=1, width=256,
                                        height=192, num_objects=4, iid_masks=True)),
                     ("synth_dense", dict(seed=9, n_gaussians=50_000, n_views=1, width=504,
                                          height=378, num_objects=8))]:
        wl = my_synth.make_workload(**kw)
        ref_scene_obj = ref.GaussianScene(means=wl.scene.means, rotations=wl.scene.rotations,
                                          scales=wl.scene.scales, opacities=wl.scene.opacities)
        ref_views = [ref.CameraView(view_id=v.view_id, width=v.width, height=v.height, fx=v.fx,
                                    fy=v.fy, cx=v.cx, cy=v.cy, world_to_camera=v.world_to_camera,
                                    near_clip=v.near_clip) for v in wl.views]
        pairs = [(rv, ref.LabelMask(rv.view_id, wl.masks[i])) for i, rv in enumerate(ref_views)]
        c = accumulate_case(ref_scene_obj, pairs, wl.num_objects, D, store_inputs=False)
        c.pop("A64")
        c["digest"] = np.frombuffer(wl.digest().encode(), dtype=np.uint8)
        c["gen_args"] = np.frombuffer(repr(sorted(kw.items())).encode(), dtype=np.uint8)
        cases[name] = c
    return cases


# ---------------------------------------------------------------- assignment
def gen_assign(acc_cases):
    rng = np.random.default_rng(4242)
    mats = {
        "rand2": (5.0 * rng.random((2, 500))).astype(np.float32),
        "rand5": rng.random((5, 300)).astype(np.float32),
        "rand16": rng.random((16, 2000), dtype=np.float32),
        "kat": np.array([[0.3, 0.5, 0.0, 0.0, 0.2, 0.1, 0.10],
                         [0.7, 0.5, 0.0, 0.4, 0.5, 0.8, 0.45]], np.float32),
        "C1": acc_cases["C1_default"]["A"],
        "C1_noisy": acc_cases["C1_noisy"]["A"],
        "synth8": acc_cases["synth_coherent"]["A"],
    }
    m = mats["rand2"]
    m[:, :40] = 0.0
    m[:, 40:60] = np.float32(1e-13)  # below UNOBSERVED_EPS in f32
    # near ties: columns whose one-vs-rest margin is within a few ulps
    t = rng.random(200).astype(np.float32)
    mats["ties"] = np.stack([t, t * np.float32(1.0000001)])
    gammas = np.array([-1.0, -0.8, -0.4, -0.25, 0.0, 0.1, 0.2, 0.4, 0.5, 0.8, 1.0])
    cases = {}
    for name, A in mats.items():
        A = np.ascontiguousarray(A, dtype=np.float32)
        out = dict(A=A, gammas=gammas)
        out["scene"] = np.stack([ref.assign_scene(ref.ContributionMatrix(A), g).membership
                                 for g in gammas])
        if A.shape[0] == 2:
            out["binary"] = np.stack([ref.assign_binary(ref.ContributionMatrix(A), g).labels
                                      for g in gammas])
        cases[name] = out
    return cases


# ---------------------------------------------------------------- rendering
def render_case(scene, view, channel, blend, member=None):
    """render_view / render_subset_alpha_depth (rasterizer.py:133-234) on one view."""
    if member is None:
        out = ref.render_view(scene, view, channel, blend)
    else:
        out = ref.render_subset_alpha_depth(scene, view, member, blend)
    c = dict(**{f"in_{a}": v for a, v in scene_arrays(scene).items()}, cam=cam_row(view),
             floors=np.array([blend.alpha_floor, blend.transmittance_floor]),
             alpha=out.alpha, depth=out.depth)
    if channel is not None:
        c["channel"] = np.asarray(channel, np.float64)
        c["value"] = out.value
    if member is not None:
        c["member"] = np.asarray(member, np.uint8)
    return c


def mask_case(scene, view, labels_or_membership, mode, tau):
    """render_binary_mask / render_scene_mask (maskrender.py:45-95)."""
    if mode == "binary":
        asn = ref.Assignment(mode="binary", gamma=0.0,
                             labels=np.asarray(labels_or_membership, np.uint8))
        out = ref.render_binary_mask(scene, asn, view, tau)
    else:
        asn = ref.Assignment(mode="scene", gamma=0.0,
                             membership=np.asarray(labels_or_membership, np.uint8))
        out = ref.render_scene_mask(scene, asn, view, tau)
    return dict(**{f"in_{a}": v for a, v in scene_arrays(scene).items()}, cam=cam_row(view),
                assignment=np.asarray(labels_or_membership, np.uint8),
                mode=np.frombuffer(mode.encode(), np.uint8), tau=np.float64(tau),
                labels=out.labels)


def iso(center, sigma, opacity):
    # reference tests/conftest.py:28-36
    return ref.Gaussian(center=np.asarray(center, np.float64), rotation=(1.0, 0.0, 0.0, 0.0),
                        scale=np.full(3, sigma), opacity=opacity)


def gen_render():
    D, X = ref.DEFAULT_BLEND, ref.EXACT_BLEND
    cases = {}
    v16 = frontal_view()
    # test_rasterizer.py:82-97 known answers
    cases["single"] = render_case(ref.GaussianScene.from_gaussians([iso((0, 0, 2.0), 0.02, 0.6)]),
                                  v16, np.array([1.0]), D)
    cases["two"] = render_case(ref.GaussianScene.from_gaussians(
        [iso((0, 0, 2.0), 0.02, 0.5), iso((0, 0, 4.0), 0.04, 0.5)]), v16, np.array([1.0, 0.0]), D)
    rng = np.random.default_rng(20240811)
    v32 = frontal_view(32, 32, 40.0)
    sc = random_scene(rng, 30)
    ch = rng.random(30)
    cases["rand_exact"] = render_case(sc, v32, ch, X)
    cases["rand_default"] = render_case(sc, v32, ch, D)
    cases["rand_nochannel"] = render_case(sc, v32, None, D)
    sc = random_scene(rng, 20)
    cases["rand_vector"] = render_case(sc, v32, rng.random((20, 3)), D)
    sc = random_scene(rng, 25)
    cases["subset"] = render_case(sc, v32, None, D, member=rng.random(25) < 0.5)
    cases["subset_empty"] = render_case(sc, v32, None, D, member=np.zeros(25, bool))
    # occluder in front must not dim the subset (test_rasterizer.py:183-191)
    sc = ref.GaussianScene.from_gaussians([iso((0, 0, 1.0), 0.02, 0.95), iso((0, 0, 3.0), 0.06, 0.7)])
    cases["subset_local"] = render_case(sc, v16, None, D, member=np.array([False, True]))
    # a denser synthetic view, ragged edge tiles, both blends
    fx = ref_synth.make_random(seed=77, n_gaussians=400, n_views=1, width=100, height=70,
                               num_objects=2)
    vw = fx.views[0]
    ch = np.random.default_rng(3).random(len(fx.scene))
    cases["synth_default"] = render_case(fx.scene, vw, ch, D)
    cases["synth_exact"] = render_case(fx.scene, vw, ch, X)
    # novel-view masks (test_maskrender.py)
    fx = ref_synth.make_two_cluster(seed=3, n_gaussians=600, n_views=8, width=96, height=96,
                                    n_mask_views=4)
    novel = fx.view(fx.heldout_view_ids()[0])
    fg = (fx.membership == 1).astype(np.uint8)
    for tau in (0.1, 0.5):
        cases[f"binary_tau{int(tau * 10)}"] = mask_case(fx.scene, novel, fg, "binary", tau)
    rng = np.random.default_rng(99)
    sc = random_scene(rng, 40)
    memb = np.zeros((4, 40), np.uint8)
    obj = rng.integers(1, 4, size=40)
    memb[obj, np.arange(40)] = 1
    memb[0] = 1 - memb[1:].max(axis=0)
    cases["scene3"] = mask_case(sc, v32, memb, "scene", 0.1)
    sc = ref.GaussianScene.from_gaussians([iso((0, 0, 2.0), 0.08, 0.9), iso((0, 0, 2.0), 0.08, 0.9)])
    cases["scene_tie"] = mask_case(sc, frontal_view(16, 16, 24.0),
                                   np.array([[0, 0], [1, 0], [0, 1]]), "scene", 0.1)
    return cases


def save(name, cases):
    flat = {}
    for case, arrays in cases.items():
        for k, v in arrays.items():
            flat[f"{case}/{k}"] = np.asarray(v)
    path = HERE / f"{name}.npz"
    np.savez_compressed(path, **flat)
    print(f"wrote {path} ({path.stat().st_size / 1e6:.2f} MB, {len(cases)} cases)")


def gen_fullres():
    """The benchmark resolution (1008 x 756, C2 camera geometry) straight from the reference:
    a 100 k-Gaussian draw of the C2 recipe, two views, E = 4 (about 35 s of reference time)."""
    D = ref.DEFAULT_BLEND
    cases = {}
    for name, kw in [("c2res_coherent", dict(seed=2, n_gaussians=100_000, n_views=2, width=1008,
                                              height=756, num_objects=4))]:
        wl = my_synth.make_workload(**kw)
        ref_scene_obj = ref.GaussianScene(means=wl.scene.means, rotations=wl.scene.rotations,
                                          scales=wl.scene.scales, opacities=wl.scene.opacities)
        ref_views = [ref.CameraView(view_id=v.view_id, width=v.width, height=v.height, fx=v.fx,
                                    fy=v.fy, cx=v.cx, cy=v.cy, world_to_camera=v.world_to_camera,
                                    near_clip=v.near_clip) for v in wl.views]
        pairs = [(rv, ref.LabelMask(rv.view_id, wl.masks[i])) for i, rv in enumerate(ref_views)]
        c = accumulate_case(ref_scene_obj, pairs, wl.num_objects, D, store_inputs=False)
        c.pop("A64")
        c["labels_g0"] = ref.assign_scene(ref.ContributionMatrix(c["A"]), 0.0).membership
        c["digest"] = np.frombuffer(wl.digest().encode(), dtype=np.uint8)
        c["gen_args"] = np.frombuffer(repr(sorted(kw.items())).encode(), dtype=np.uint8)
        cases[name] = c
        # novel-view rendering at the same resolution: render_view with a
        # scalar channel on view 0 (20 000 sampled pixels + whole-image sums), and
        # render_scene_mask of the reference's own labels on view 1 (all pixels)
        t0 = time.perf_counter()
        ch = np.random.default_rng(5).random(len(wl.scene))
        out = ref.render_view(ref_scene_obj, ref_views[0], ch, D)
        idx = np.sort(np.random.default_rng(6).choice(out.alpha.size, 20_000, replace=False))
        cases[name + "_render"] = dict(  # channel = default_rng(5).random(N), not stored
            idx=idx, alpha=out.alpha.ravel()[idx], depth=out.depth.ravel()[idx],
            value=out.value.ravel()[idx],
            sums=np.array([out.alpha.sum(), out.depth.sum(), out.value.sum()]))
        asn = ref.Assignment(mode="scene", gamma=0.0, membership=c["labels_g0"])
        m = ref.render_scene_mask(ref_scene_obj, asn, ref_views[1], 0.5)
        cases[name + "_mask"] = dict(labels=m.labels, tau=np.float64(0.5))
        print(f"  render + scene mask 1008x756: {time.perf_counter() - t0:.1f}s", flush=True)
    return cases


def gen_scene_ply(tmpdir):
    """Splat checkpoints loaded by the reference's own load_scene_ply (ply.py:63-106):
    the file bytes and the activated float64 arrays.  The
    second file interleaves extra per-vertex properties (f_rest_*, a non-standard
    order) so a loader must honour the header's property offsets."""
    from splatlift import ply as ref_ply
    cases = {}
    rng = np.random.default_rng(31)
    n = 3000
    base = dict(x=rng.normal(size=n), y=rng.normal(size=n), z=rng.uniform(2, 6, n),
                nx=np.zeros(n), ny=np.zeros(n), nz=np.zeros(n),
                f_dc_0=rng.normal(size=n), f_dc_1=rng.normal(size=n), f_dc_2=rng.normal(size=n),
                opacity=rng.normal(0, 3, n), scale_0=rng.uniform(-7, 1, n),
                scale_1=rng.uniform(-7, 1, n), scale_2=rng.uniform(-7, 1, n),
                rot_0=rng.normal(size=n), rot_1=rng.normal(size=n), rot_2=rng.normal(size=n),
                rot_3=rng.normal(size=n))
    # extreme but valid values: opacity logits far out, near-degenerate quaternions
    base["opacity"][:4] = [40.0, -40.0, 700.0, -700.0]
    base["rot_1"][4:8] = base["rot_2"][4:8] = base["rot_3"][4:8] = 0.0
    base["rot_0"][4:8] = [1e-30, 3e-38, 2.0, -1.0]
    layouts = {
        "plain": list(ref_ply.REQUIRED_PROPERTIES),
        "interleaved": (["f_rest_0", "rot_3", "x", "f_rest_1", "scale_2", "opacity"] +
                        [p for p in ref_ply.REQUIRED_PROPERTIES
                         if p not in ("rot_3", "x", "scale_2", "opacity")] + ["f_rest_2"]),
    }
    for name, props in layouts.items():
        rec = np.zeros(n, dtype=np.dtype([(p, "<f4") for p in props]))
        for p in props:
            rec[p] = base[p] if p in base else rng.normal(size=n)
        path = Path(tmpdir) / f"{name}.ply"
        head = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
        head += [f"property float {p}" for p in props] + ["end_header"]
        with open(path, "wb") as fh:
            fh.write(("\n".join(head) + "\n").encode("ascii"))
            rec.tofile(fh)
        sc = ref_ply.load_scene_ply(path)
        cases[name] = dict(ply=np.frombuffer(path.read_bytes(), dtype=np.uint8),
                           means=sc.means, rotations=sc.rotations, scales=sc.scales,
                           opacities=sc.opacities, colors=sc.colors_dc)
    return cases


def fixture_case(fix, pairs=None):
    """Inputs of a reference SynthFixture's training views, verbatim."""
    pairs = fix.training_views() if pairs is None else pairs
    out = {f"in_{a}": c for a, c in scene_arrays(fix.scene).items()}
    out["cams"] = np.stack([cam_row(v) for v, _ in pairs])
    out["masks"] = np.stack([m.labels for _, m in pairs])
    return out


def gen_acceptance():
    """Inputs and reference answers for the acceptance suite restated on the GPU
    (tests/test_gpu_acceptance.py): reference tests/test_acceptance.py:53-77
    (global optimality vs the exhaustive oracle, 200 seeded instances),
    :140-197 (gamma nesting, scale invariance, scene/binary consistency),
    :230-247 (latency fixture) and tests/test_solver.py:100-159."""
    from splatlift import brute_force_oracle, objective_value
    from splatlift.synth import make_random, make_two_cluster
    X = ref.EXACT_BLEND
    cases = {}
    t0 = time.perf_counter()
    master = np.random.default_rng(1234)  # test_acceptance.py:56-66, same draws
    for case in range(200):
        seed = int(master.integers(0, 2**31))
        fix = make_random(seed=seed, n_gaussians=int(master.integers(4, 13)),
                          n_views=int(master.integers(1, 4)), width=int(master.integers(8, 17)),
                          height=int(master.integers(8, 17)))
        pairs = fix.training_views()
        c = fixture_case(fix, pairs)
        matrix = ref.accumulate_contributions(fix.scene, pairs, 2, X)
        labels = ref.assign_binary(matrix, 0.0).labels
        best_labels, best = brute_force_oracle(fix.scene, pairs, X)
        c.update(A=matrix.values, labels=labels, best_labels=best_labels,
                 best=np.float64(best),
                 achieved=np.float64(objective_value(fix.scene, pairs, labels, X)))
        cases[f"opt{case:03d}"] = c
    print(f"  optimality instances: {time.perf_counter() - t0:.1f}s", flush=True)
    for case in range(5):  # test_acceptance.py:146-150
        fix = make_random(seed=900 + case, n_gaussians=40, n_views=2, width=24, height=24)
        cases[f"mono{case}"] = fixture_case(fix)
    for case in range(20):  # test_acceptance.py:176-180
        e = 3 + case % 3
        fix = make_random(seed=500 + case, n_gaussians=20, n_views=2, width=16, height=16,
                          num_objects=e)
        c = fixture_case(fix)
        c["E"] = np.int64(e)
        cases[f"rel{case:02d}"] = c
    for seed in range(6):  # test_solver.py:115-118
        fix = make_random(seed=seed, n_gaussians=15, n_views=2, width=16, height=16,
                          num_objects=4)
        c = fixture_case(fix)
        c["E"] = np.int64(4)
        cases[f"solver_rel{seed}"] = c
    fix = make_two_cluster(seed=42, n_gaussians=2000, n_views=12, width=128, height=128,
                           n_mask_views=6)  # test_acceptance.py:47-51
    c = fixture_case(fix)
    c["A"] = ref.accumulate_contributions(fix.scene, fix.training_views(), 2).values
    cases["cluster"] = c
    return cases


def gen_fuzz(seeds=None, budget_s=240.0):
    """The reference's own outputs on the adversarial fuzz cases of
    tests/fuzz_cases.py (inputs regenerated at test time, pinned by digest):
    A (float32 and float64), assign_scene membership / assign_binary labels at
    the case's gamma, and render_view (alpha, depth; a 3-channel property composited alongside) plus
    render_scene_mask of the first view."""
    sys.path.insert(0, str(ROOT / "tests"))
    import fuzz_cases as fz
    from splatlift import maskrender as ref_mask
    from splatlift import rasterizer as ref_rast
    from splatlift import solver as ref_solver

    cases, spent = {}, 0.0
    for seed in (seeds if seeds is not None else range(fz.N_CASES)):
        c = fz.case_arrays(seed)
        n = len(c["opac"])
        px = sum(int(r[0]) * int(r[1]) for r in c["cams"])
        if n * px > 4e8 or n * c["E"] > 25000:  # fixture size and reference time
            continue
        t0 = time.perf_counter()
        scene = ref_scene.GaussianScene(c["means"], c["quats"], c["scales"], c["opac"])
        views = [ref_scene.CameraView(view_id=i, width=int(r[0]), height=int(r[1]), fx=r[2],
                                      fy=r[3], cx=r[4], cy=r[5], world_to_camera=r[7:].reshape(4, 4),
                                      near_clip=r[6]) for i, r in enumerate(c["cams"])]
        pairs = [(v, ref_contrib.LabelMask(v.view_id, m)) for v, m in zip(views, c["masks"])]
        blend = ref.BlendConfig(*c["floors"])
        out = accumulate_case(scene, pairs, c["E"], blend, store_inputs=False)
        del out["A64"]  # the reference's float32 matrix is the fixture
        M = ref_contrib.ContributionMatrix(out["A"])
        out["membership"] = ref_solver.assign_scene(M, c["gamma"]).membership.astype(np.uint8)
        if c["E"] == 2:
            out["labels"] = ref_solver.assign_binary(M, c["gamma"]).labels.astype(np.uint8)
        ch, memb, tau = fz.render_extras(seed, n, c["E"])
        if views[0].width * views[0].height <= 6000:  # render fixtures of the small views
            r = ref_rast.render_view(scene, views[0], ch, blend)
            out.update(r_alpha=r.alpha, r_depth=r.depth)
            asn = ref_solver.Assignment(mode="scene", gamma=0.0, membership=memb.astype(bool))
            out["r_mask"] = ref_mask.render_scene_mask(scene, asn, views[0], tau, blend).labels
        out["digest"] = np.frombuffer(fz.digest(c).encode(), np.uint8)
        cases[f"s{seed}"] = out
        spent += time.perf_counter() - t0
        print(f"  fuzz seed {seed}: N={n} px={px} E={c['E']} {time.perf_counter() - t0:.1f}s",
              flush=True)
        if spent > budget_s:
            break
    return cases


def main(which=None):
    if which == "fuzz":
        save("fuzz", gen_fuzz())
        return
    if which == "fullres":
        save("accumulate_fullres", gen_fullres())
        return
    if which == "acceptance":
        save("acceptance", gen_acceptance())
        return
    if which == "ply":
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            save("scene_ply", gen_scene_ply(d))
        return
    if which in (None, "render"):
        save("render", gen_render())
    if which == "render":
        return
    save("projection", gen_projection())
    save("binning", gen_binning())
    acc = gen_accumulate()
    save("accumulate", acc)
    save("assign", gen_assign(acc))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
