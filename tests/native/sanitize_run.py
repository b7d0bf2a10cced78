"""Small end-to-end run of every product kernel for compute-sanitizer
(memcheck): fused K1 (both variants, host and device frames, evaluation
epilogue), per-bank kernels, Augmented4, registration + dilation, fusion,
per-pixel API, plane gather/scatter.  Exit 0 when all results match the
oracle (TEST INFRASTRUCTURE)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import paper_2110_14934_b200 as R  # noqa: E402
from helpers import holes, random_rig  # noqa: E402

port = O.Port()
w, h, S = 45, 30, 2
for variant in ("ldg", "auto"):
    proc = R.SequenceProcessor(w, h, R.RunConfig.defaults(), streams=S, variant=variant)
    orc = [O.PortProcessor(port, w * h, O.depth_cfg(3, learning_rate=0.05, initial_sigma=15.0),
                           O.depth_cfg(3)) for _ in range(S)]
    scenes = [O.PortScene(port, "A", w, h, seed=s + 1) for s in range(S)]
    for f in range(6):
        frs = [sc.render(f) for sc in scenes]
        r, g, b = (np.stack([getattr(x, k) for x in frs]) for k in ("r", "g", "b"))
        d = np.stack([holes(x.depth, f) for x in frs])
        gt = np.stack([x.gt for x in frs])
        fm = proc.process(r, g, b, d, gt=gt)
        for s in range(S):
            _, _, fu = orc[s].process(r[s], g[s], b[s], d[s])
            assert np.array_equal(fm.fused[s].ravel(), fu)
a = random_rig(np.random.default_rng(1), w, h)
rig = R.CameraRig()
rig.depth_cam, rig.color_cam = list(a[0:4]), list(a[4:8])
rig.rotation, rig.translation_mm, rig.depth_scale = list(a[8:17]), list(a[17:20]), float(a[20])
up = R.SequenceProcessor(w, h, R.RunConfig.defaults(), rig=rig, registered=False)
for f in range(4):
    fr = O.PortScene(port, "A", w, h).render(f)
    up.process(fr.r, fr.g, fr.b, fr.depth, gt=fr.gt)
bank = R.ModelBank(w, h, "Augmented4", R.MixtureConfig(components=4))
for f in range(3):
    fr = O.PortScene(port, "B", w, h).render(f)
    R.segment_augmented(bank, fr.r, fr.g, fr.b, fr.depth, R.DepthRescale(), R.MixtureConfig(components=4))
bank.upload_plane(0, bank.mean_plane(0, 0))
print(R.confusion_counts(np.ones((3, 5), np.uint8), np.zeros((3, 5), np.uint8)))
mix = R.init_mixture([1.0, 2.0, 3.0], R.MixtureConfig())
R.step_pixel(mix, [1.0, 2.0, 3.0], R.MixtureConfig())
print("sanitize_run ok")
