"""SASS evidence for the tcgen05 / TMA path: per-kernel counts of the Blackwell instructions in
paper_2509_24006_b200/libsla_b200.so (cuobjdump -sass, names demangled with c++filt).

    python profiles/sass_counts.py [out.md]     (no GPU needed)
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2509_24006_b200", "libsla_b200.so")
COLS = [("UTCHMMA", "tcgen05.mma"), ("UTCBAR", "tcgen05.commit"), ("UTMALDG", "TMA load"),
        ("UTMASTG", "TMA store"), ("LDTM", "tcgen05.ld"), ("STTM", "tcgen05.st"),
        ("UTCATOMSWS", "TMEM alloc/dealloc"), ("ELECT", "elect.sync")]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_sass.md")
    sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
    rows = []
    for part in re.split(r"\n\s*Function : ", sass)[1:]:
        mangled = part.split("\n", 1)[0].strip()
        name = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"slab::\(anonymous namespace\)::|slab::", "", name)
        name = re.sub(r"\(.*\)$", "", name).replace("__nv_bfloat16", "bf16")
        ops = collections.Counter(re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", part))
        if not any(ops[c] for c, _ in COLS[:6]):
            continue
        mc = len(re.findall(r"UTMALDG\S*MULTICAST|\.MULTICAST", part))
        rows.append((name, [ops[c] for c, _ in COLS], mc))
    rows.sort()
    with open(out, "w") as f:
        f.write("# SASS evidence: Blackwell tcgen05 / TMA instructions per kernel\n\n")
        f.write("`python profiles/sass_counts.py` over `cuobjdump -sass libsla_b200.so` (static counts per kernel "
                "instance; generic SIMT and diagnostic kernels without tcgen05/TMA omitted).\n\n")
        f.write("| kernel | " + " | ".join(f"{c} ({d})" for c, d in COLS) + " | multicast (TMA + commit) |\n")
        f.write("|---|" + "---|" * (len(COLS) + 1) + "\n")
        for name, cnt, mc in rows:
            f.write(f"| `{name}` | " + " | ".join(str(x) for x in cnt) + f" | {mc} |\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
