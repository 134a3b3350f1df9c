"""Markdown tables of the measured parity errors logged by the -m gpu tests ($SLA_PARITY_LOG).

  python profiles/parity_table.py profiles/r02_parity_errors.jsonl   # scale cases (vs the reference)
  python profiles/parity_table.py profiles/r02_parity_small.jsonl    # small-shape tests (worst per test)
"""
import collections
import json
import sys


def scale(rows):
    keys = ("o", "o_s", "o_l", "dq_total", "dk_total", "dv", "dw")
    print("| case | head | label flips | " + " | ".join(keys) + " | lse max-abs |")
    print("|---|---|---|" + "---|" * len(keys) + "---|")
    for r in rows:
        cells = [f"{r[k]['rel']:.2e} ({r[k]['bf16_floor']:.1e})" if r[k]["bf16_floor"] else f"{r[k]['rel']:.2e}"
                 for k in keys]
        print(f"| {r['case']} | {r['head']} | {r['label_flips']} | " + " | ".join(cells) + f" | {r['lse']['max_abs']:.1e} |")
    print("\nrel_diff (floor 1.0) against the reference's f32 result; in brackets the rel_diff of the "
          "reference's own result rounded to bf16 (the storage floor of a bf16 output).")


def small(rows):
    worst, tol = collections.defaultdict(float), {}
    for x in rows:
        if "test" not in x:
            continue
        k = (x["test"].split("[")[0].split("::")[-1], x["key"])
        worst[k] = max(worst[k], x["err"])
        tol[k] = x["tol"]
    print("| test | tensor | worst measured | gate |\n|---|---|---|---|")
    for k in sorted(worst):
        print(f"| {k[0]} | {k[1]} | {worst[k]:.2e} | {tol[k]:.0e} |")


if __name__ == "__main__":
    rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
    if sys.argv[2:] == ["scale"] or (rows and all("case" in r for r in rows)):
        scale([r for r in rows if "case" in r])
    else:
        small(rows)
