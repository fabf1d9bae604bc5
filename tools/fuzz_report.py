"""Adversarial fuzz parity summary (GPU): every case of tests/fuzz_cases.py through
the public API against the oracle, and -- where tests/golden/fuzz.npz has them --
against the reference's own outputs.  Writes gpurun_out/fuzz_parity.json.

    PYTHONPATH=.:tests python tools/fuzz_report.py
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, "tests")
import oracle  # noqa: E402
from conftest import cam_from_row, load_golden  # noqa: E402
from fuzz_cases import N_CASES, ambiguous_mask_pixels, case_arrays, label_band, render_extras  # noqa: E402

from paper_2409_08270_b200 import (Assignment, BlendConfig, ContributionMatrix, GaussianScene,  # noqa: E402
                                   LabelMask, accumulate_contributions, assign_scene,
                                   render_scene_mask, render_view)


def main():
    ref_all = load_golden("fuzz")
    agg = dict(cases=0, entries=0, vs_oracle_entries_differing=0, vs_oracle_max_rel=0.0,
               vs_reference_cases=0, vs_reference_entries=0, vs_reference_entries_differing=0,
               vs_reference_max_rel=0.0, label_flips_vs_reference=0,
               label_flips_outside_band=0, band_size=0, render_views=0,
               render_alpha_max_rel_vs_oracle=0.0, mask_pixels=0, mask_pixels_differing_vs_oracle=0,
               mask_pixels_ambiguous=0, mask_differing_outside_ambiguous=0, fixed_cases=0,
               f64_cases=0)
    t0 = time.time()
    for seed in range(N_CASES):
        c = case_arrays(seed)
        scene = GaussianScene(c["means"], c["quats"], c["scales"], c["opac"])
        views = [cam_from_row(r, i) for i, r in enumerate(c["cams"])]
        pairs = [(v, LabelMask(v.view_id, m)) for v, m in zip(views, c["masks"])]
        blend = BlendConfig(*c["floors"])
        E, g = c["E"], c["gamma"]
        fixed = blend.alpha_floor * blend.transmittance_floor >= 2.0 ** -26
        agg["fixed_cases" if fixed else "f64_cases"] += 1
        A = accumulate_contributions(scene, pairs, E, blend).values
        ref = oracle.accumulate(scene.means, scene.rotations, scene.scales, scene.opacities,
                                [oracle.camera_of(v) for v in views], c["masks"], E,
                                *c["floors"], threads=8, as_float32=False)
        agg["cases"] += 1
        agg["entries"] += A.size
        agg["vs_oracle_entries_differing"] += int(np.count_nonzero(A != ref.astype(np.float32)))
        rel = np.abs(A - ref) / np.maximum(np.abs(ref), 1e-30)
        agg["vs_oracle_max_rel"] = max(agg["vs_oracle_max_rel"], float(np.where(ref != 0, rel, 0).max(initial=0)))
        r = ref_all.get(f"s{seed}")
        if r is not None:
            agg["vs_reference_cases"] += 1
            agg["vs_reference_entries"] += A.size
            agg["vs_reference_entries_differing"] += int(np.count_nonzero(A != r["A"]))
            rr = np.abs(A.astype(np.float64) - r["A"]) / np.maximum(np.abs(r["A"]), 1e-30)
            agg["vs_reference_max_rel"] = max(agg["vs_reference_max_rel"],
                                              float(np.where(r["A"] != 0, rr, 0).max(initial=0)))
            memb = assign_scene(ContributionMatrix(A), g).membership
            flips = (memb != r["membership"]).any(axis=0)
            band = label_band(oracle, r["A"], g, True)
            agg["label_flips_vs_reference"] += int(flips.sum())
            agg["label_flips_outside_band"] += int((flips & ~band).sum())
            agg["band_size"] += int(band.sum())
        if seed % 2 == 0:
            ch, memb, tau = render_extras(seed, len(scene), E)
            for v in views:
                o = oracle.camera_of(v)
                out = render_view(scene, v, ch, blend)
                _, alpha, _ = oracle.render_view(scene.means, scene.rotations, scene.scales,
                                                 scene.opacities, o, ch, None, *c["floors"])
                agg["render_views"] += 1
                agg["render_alpha_max_rel_vs_oracle"] = max(
                    agg["render_alpha_max_rel_vs_oracle"],
                    float((np.abs(out.alpha - alpha) / np.maximum(alpha, 1e-300)).max(initial=0)))
                got = render_scene_mask(scene, Assignment(mode="scene", gamma=0.0, membership=memb),
                                        v, tau, blend).labels
                want = oracle.render_mask(scene.means, scene.rotations, scene.scales,
                                          scene.opacities, o, memb, tau, *c["floors"])
                amb = ambiguous_mask_pixels(oracle, scene.means, scene.rotations, scene.scales,
                                            scene.opacities, o, memb, tau, c["floors"])
                d = got != want
                agg["mask_pixels"] += d.size
                agg["mask_pixels_differing_vs_oracle"] += int(d.sum())
                agg["mask_pixels_ambiguous"] += int(amb.sum())
                agg["mask_differing_outside_ambiguous"] += int((d & ~amb).sum())
    agg["seconds"] = round(time.time() - t0, 1)
    agg["source"] = "tools/fuzz_report.py over tests/fuzz_cases.py (160 seeded adversarial cases)"
    print(json.dumps(agg, indent=1))
    with open("gpurun_out/fuzz_parity.json", "w") as f:
        json.dump(agg, f, indent=1)


if __name__ == "__main__":
    main()
