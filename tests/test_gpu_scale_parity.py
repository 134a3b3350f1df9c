"""Parity of the tcgen05 path against the REFERENCE ITSELF at the benchmarked shapes.

The reference's unmodified C++ library (oracle/_ref/libsla_ref.so, built by oracle/Makefile
from /root/reference/proj/core and shipped with the repo snapshot) runs the reference's own
call sequence -- sla_forward -> combine_outputs -> proj_backward -> sla_backward, f32,
threads = all host cores (forward.cpp:174-185, backward.cpp:12-216, the acceptance sweep of
acceptance_main.cpp:51-102) -- on the same bf16-exact SplitMix64 inputs the GPU gets.

Cases:
  c3_softmax / c3_elu1  N = 32768, d = 128, 2 heads, k_h 5 %, dynamic mask   (T = 512, n1 = 26)
  c4_kh20               N = 32768, 1 head, k_h 20 %                          (n1 = 102)
  c5_unit               N = 75648, 1 head, k_h 5 %  (T = 1182 > 512: block-per-row classifier, n1 = 59)
  rescale               N = 32768, 1 head, scores rising along the key axis, so the forward's
                        lazy online-softmax rescale (running max up by > 2^8) fires on most rows

Labels must be bit-identical to the reference's.  Outputs and gradients are gated on
rel_diff (floor 1.0, mat.hpp:169-178) and max-abs; the gates are ~2-3x the errors measured on
B200 (table "measured parity at scale"), and every run appends its
measured errors to $SLA_PARITY_LOG (JSON lines) when that is set.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2509_24006_b200 import SLA, SlaConfig

pytestmark = pytest.mark.gpu

TENSORS = ("o", "o_s", "o_l", "dq_total", "dk_total", "dv", "dw")
# gates: rel_diff (floor 1.0) per tensor; lse max-abs on live rows.  Measured on B200
# (profiles/r02_parity_errors.jsonl): worst over the iid cases o 1.4e-3,
# o_l 1.1e-4, dq_total 2.3e-3, dk_total 2.3e-3, dv 1.3e-3, dw 2.3e-3, lse 1.9e-6 -- each within
# ~2.5x of the error of merely storing the reference's f32 result in bf16.  Gates are ~2-3x those.
GATE = {"o": 4e-3, "o_s": 4e-3, "o_l": 3e-4, "dq_total": 5e-3, "dk_total": 5e-3, "dv": 3.5e-3,
        "dw": 6e-3, "lse": 5e-6}
# the rescale case drives scores to |S| ~ 20 (sharper softmax rows: larger bf16 P rounding);
# measured o 4.5e-3, o_l 3.1e-4, dq_total 5.5e-3, dk_total 4.4e-3, dv 3.0e-3, lse 1.1e-5
GATE_RESCALE = {"o": 1e-2, "o_s": 1e-2, "o_l": 8e-4, "dq_total": 1.2e-2, "dk_total": 1e-2, "dv": 7e-3,
                "dw": 7e-3, "lse": 3e-5}


def _bf(a):
    return O.to_bf16_exact(a)


def _inputs(case, n, d, heads, seed):
    rng = O.Rng(seed)
    xs = []
    for _ in range(heads):
        x = dict(q=rng.gaussian(n, d), k=rng.gaussian(n, d), v=rng.gaussian(n, d), do=rng.gaussian(n, d))
        if case == "rescale":
            # key block j scaled by 0.25 + 1.75 j / T and queries by 3: the scores of a row grow
            # along its ascending critical list, so its running max climbs by > 8 (log2 units)
            t = n // 64
            ramp = np.repeat(0.25 + 1.75 * np.arange(t) / t, 64)[:, None]
            x["k"] = x["k"] * ramp
            x["q"] = x["q"] * 3.0
        xs.append({nm: _bf(a) for nm, a in x.items()})
    w = _bf(rng.gaussian(d, d, 0.1))
    return xs, w


def _rescale_rows(q, k, labels, scale_log2, thresh=8.0):
    """Rows whose running max (log2 units, ascending critical list) grows by > thresh after the
    first tile -- the kernel's lazy-rescale condition (attn_fwd.cu, `need`)."""
    t_m = labels.shape[0]
    hits = 0
    for i in range(t_m):
        cols = np.nonzero(labels[i] == 1)[0]
        if cols.size < 2:
            continue
        qi = q[i * 64:(i + 1) * 64].astype(np.float32)
        kc = np.concatenate([k[j * 64:(j + 1) * 64] for j in cols]).astype(np.float32)
        s = (qi @ kc.T) * scale_log2                      # [64, 64 * len(cols)]
        tile_max = s.reshape(64, cols.size, 64).max(axis=2)  # [64, tiles]
        m_used = tile_max[:, 0].copy()
        for tt in range(1, cols.size):
            m_new = np.maximum(m_used, tile_max[:, tt])
            need = m_new > m_used + thresh
            hits += int(need.sum())
            m_used = np.where(need, m_new, m_used)
    return hits


def _T(a):
    return torch.tensor(np.array(a), dtype=torch.float32).to("cuda", torch.bfloat16).contiguous()


CASES = {
    #              n      d   heads  k_h   k_l   phi        seed
    "c3_softmax": (32768, 128, 2, 5.0, 10.0, "softmax", 101),
    "c3_elu1": (32768, 128, 2, 5.0, 10.0, "elu1", 202),
    "c4_kh20": (32768, 128, 1, 20.0, 10.0, "softmax", 303),
    "c5_unit": (75648, 128, 1, 5.0, 10.0, "softmax", 404),
    "rescale": (32768, 128, 1, 5.0, 10.0, "softmax", 505),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_scale_parity_against_reference(case):
    if not O.Reference.available():
        pytest.fail("oracle/_ref/libsla_ref.so missing: run __graft_entry__.build() where /root/reference exists")
    n, d, heads, k_h, k_l, phi, seed = CASES[case]
    xs, w = _inputs(case, n, d, heads, seed)
    cfg = SlaConfig(k_h=k_h, k_l=k_l, phi=phi)
    op = SLA(1, heads, n, d, 64, 64, cfg, torch.bfloat16)
    assert op.path == "tcgen05"
    q, k, v, do = (_T([[x[nm] for x in xs]]) for nm in ("q", "k", "v", "do"))
    wt = _T([w] * heads)
    st = op.forward(q, k, v, wt)
    g = op.backward(st, q, k, v, wt, do)
    torch.cuda.synchronize()
    threads = os.cpu_count() or 1
    log = os.environ.get("SLA_PARITY_LOG")
    worst = {}
    for h, x in enumerate(xs):
        ref = O.Reference.run(x["q"], x["k"], x["v"], 64, 64, k_h, k_l, phi, threads=threads, w=w,
                              d_out=x["do"], dtype=np.float32)
        lab = st.labels[0, h].cpu().numpy()
        flips = int((lab != ref["labels"]).sum())
        got = {"o": st.o[0, h], "o_s": st.o_s[0, h], "o_l": st.o_l[0, h], "dq_total": g.dq_total[0, h],
               "dk_total": g.dk_total[0, h], "dv": g.dv[0, h], "dw": g.dproj[h]}
        row = {"case": case, "head": h, "n": n, "d": d, "k_h": k_h, "phi": phi, "label_flips": flips}
        for nm in TENSORS:
            a = got[nm].double().cpu().numpy()
            b = ref[nm].astype(np.float64)
            # bf16 floor: the error of merely storing the reference's f32 result in bf16
            floor = O.rel_diff(_bf(b), b, 1.0) if nm != "dw" else 0.0
            row[nm] = {"rel": O.rel_diff(a, b, 1.0), "max_abs": float(np.abs(a - b).max()),
                       "bf16_floor": floor, "ref_max": float(np.abs(b).max())}
        lse = st.lse[0, h].cpu().numpy().astype(np.float64)
        rl = ref["lse"].astype(np.float64)
        live = rl > -1e29
        assert (lse[~live] == np.float32(-1e30)).all()
        row["lse"] = {"max_abs": float(np.abs(lse[live] - rl[live]).max()) if live.any() else 0.0}
        if case == "rescale":
            row["rescale_rows"] = _rescale_rows(x["q"], x["k"], lab, np.log2(np.e) / np.sqrt(d))
        if log:
            with open(log, "a") as f:
                f.write(json.dumps(row) + "\n")
        assert flips == 0, f"{case} head {h}: {flips} labels differ from the reference"
        for nm in TENSORS:
            worst[nm] = max(worst.get(nm, 0.0), row[nm]["rel"])
        worst["lse"] = max(worst.get("lse", 0.0), row["lse"]["max_abs"])
        if case == "rescale":
            assert row["rescale_rows"] > 0, "the lazy-rescale path was not exercised"
    gate = GATE_RESCALE if case == "rescale" else GATE
    bad = {nm: v for nm, v in worst.items() if v > gate[nm]}
    assert not bad, f"{case}: over the gate {bad} (gates {gate})"
