"""Generates tests/golden/fullsize_cfg{1,3}.npz: the UNMODIFIED reference
(oracle/_ref, fp64, all host cores) run on BASELINE configs 1 and 3 at their
stated sizes and full schedules (config 1: 160x192x224, 200/100/50, LNCC
kernel 5; config 3: 192x192x208, 250/150/75, SSD, sigma_grad 1.5) — several
minutes of CPU each, so it is run once here and committed:

    make -C oracle ref && python tests/golden/make_golden_fullsize.py [1] [3]

Stored (small): sha256 of the fp32 input volumes (the GPU test regenerates
them with paper_2404_01249_b200.synth and refuses to compare if they differ),
every iteration's loss and max step, final loss / singularity fraction, the
reference's warped-label overlap (MO mean, MO Klein), and the final field at
every 4th voxel per axis (fp64) for the fp64-context field criterion.

It also runs the same unmodified reference built with FMA contraction
(oracle/_ref/libdifform_ref_fma.so, `make -C oracle ref-fma`): an IEEE-valid
rounding change of the reference itself.  Its divergence from the plain build
(per-iteration loss, field) is stored as the conditioning envelope of the
loop on this input.
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle  # noqa: E402
from paper_2404_01249_b200 import synth  # noqa: E402

STRIDE = 4


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(config: int):
    ref = pyoracle.reference()
    t0 = time.time()
    p = synth.make_pair(config, seed=0)
    t1 = time.time()
    fld, log = ref.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    t2 = time.time()
    w = ref.warp_labels(p.grid, p.moving_labels, fld)
    mo, klein = ref.overlap_dice(p.grid, w, p.fixed_labels)
    mo0, _ = ref.overlap_dice(p.grid, p.moving_labels, p.fixed_labels)
    t3 = time.time()
    ffma, lfma = pyoracle.reference_fma().register_images(p.grid, p.fixed, p.moving, p.config,
                                                          p.schedule)
    t4 = time.time()
    lf = np.array([r.loss for r in lfma.iterations])
    out = os.path.join(HERE, f"fullsize_cfg{config}.npz")
    np.savez_compressed(
        out, fixed_sha=np.array(sha(p.fixed)), moving_sha=np.array(sha(p.moving)),
        labels_sha=np.array(sha(p.moving_labels)),
        losses=np.array([r.loss for r in log.iterations]),
        max_steps=np.array([r.max_step for r in log.iterations]),
        scale_index=np.array([r.scale_index for r in log.iterations]),
        final_loss=np.array(log.final_loss), sing=np.array(log.final_singularity_fraction),
        dice_mo=np.array(mo), dice_klein=np.array(klein), dice_identity=np.array(mo0),
        field_sub=fld[::STRIDE, ::STRIDE, ::STRIDE].copy(), stride=np.array(STRIDE),
        ref_seconds=np.array(t2 - t1), threads=np.array(os.cpu_count()),
        fma_losses=lf, fma_field_sub=ffma[::STRIDE, ::STRIDE, ::STRIDE].copy(),
        fma_field_maxdiff=np.array(np.abs(ffma - fld).max()), fma_seconds=np.array(t4 - t3))
    print(f"config {config}: inputs {t1 - t0:.1f} s, reference register_images {t2 - t1:.1f} s, "
          f"{len(log.iterations)} records, final loss {log.final_loss:.6f}, "
          f"dice {mo0:.4f} -> {mo:.4f}; FMA build: loss rel max "
          f"{(np.abs(lf - np.array([r.loss for r in log.iterations])) / np.abs(lf)).max():.2e}, "
          f"field max {np.abs(ffma - fld).max():.3e}; wrote {out}", flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["1", "3"]):
        run(int(c))
