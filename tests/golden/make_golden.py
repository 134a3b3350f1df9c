"""Generate the golden fixtures from the REFERENCE ITSELF (oracle/_ref/libsla_ref.so, built
by oracle/Makefile from the unmodified sources under /root/reference/proj/core).

Inputs are not stored: they are regenerated bit-exactly from SplitMix64 seeds
(rng.hpp:22-64) by tests/_cases.py.  Only the reference's outputs are stored.

    python tests/golden/make_golden.py        # needs /root/reference (this container only)
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as O  # noqa: E402
import _cases as cases  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    O.build(ref=True)
    assert O.Reference.available(), "oracle/_ref not built (needs /root/reference)"
    R = O.Reference

    # 1) small training steps, f64 and f32 reference paths, injected random masks
    small = {}
    for c in cases.SMALL:
        x = cases.small_inputs(c)
        dts = ((np.float64, "f64"), (np.float32, "f32")) if c["d"] <= 16 else ((np.float32, "f32"),)
        for dt, tag in dts:
            r = R.run(x["q"], x["k"], x["v"], c["b"], c["b"], phi_kind=c["phi"], w=x["w"],
                      labels=x["labels"], d_out=x["do"], dtype=dt)
            for key in ("o", "o_s", "o_l", "lse", "dq_total", "dk_total", "dv", "dw"):
                small[f"{c['name']}/{tag}/{key}"] = r[key]
    np.savez_compressed(os.path.join(OUT, "small_steps.npz"), **small)

    # 2) C1 (BASELINE configs[0]): dynamic mask, f32 reference on bf16-exact inputs
    c1 = {}
    for h in range(cases.C1["heads"]):
        x = cases.c1_inputs(h)
        r = R.run(x["q"], x["k"], x["v"], 64, 64, k_h=5.0, k_l=10.0, phi_kind=cases.C1["phi"],
                  w=x["w"], d_out=x["do"], dtype=np.float32, threads=os.cpu_count())
        keys = ("labels", "o", "lse", "dq_total", "dk_total", "dv", "dw") if h == 0 else ("labels", "lse")
        for key in keys:
            c1[f"h{h}/{key}"] = r[key]
    np.savez_compressed(os.path.join(OUT, "c1_step.npz"), **c1)

    # 3) masks at the Wan2.1 shape (N=32768, d=128, T=512): iid and peaked inputs
    masks = {}
    for name, (seed, peaked) in cases.C2_MASKS.items():
        q, k = cases.c2_qk(seed, peaked)
        p_c = R.predict(q, k, 64, 64)
        masks[f"{name}/labels"] = R.classify(p_c, 5.0, 10.0)
        # smallest relative gap at the critical boundary, for the near-tie report
        srt = -np.sort(-p_c, axis=1)
        masks[f"{name}/gap_crit"] = (srt[:, 25] - srt[:, 26]) / srt[:, 25]
    np.savez_compressed(os.path.join(OUT, "c2_masks.npz"), **masks)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
