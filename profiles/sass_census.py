"""Per-kernel SASS instruction census of the built engine (runs here, no GPU): the evidence that the
hot kernels run on the Blackwell-native paths - UTCHMMA / UTCIMMA (tcgen05.mma kind::f16 / kind::i8,
".2CTA" = cta_group::2), UTCCP (tcgen05.cp), UTMALDG / UTMASTG (TMA loads / stores), UTMAREDG (TMA
reduce), LDTM (tcgen05.ld) - versus HMMA (mma.sync) and MUFU (SFU) ops.

    python profiles/sass_census.py            # -> profiles/r02_sass_census.json + .md
"""
from __future__ import annotations

import json
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "paper_2507_04967_b200" / "libiolm_cuda.so"
OPS = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "UTCCP", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "LDTM", "STTM",
       "HMMA", "IMMA", "MUFU.EX2", "MUFU.TANH", "MUFU.RCP", "SYNCS", "ELECT"]


def demangle(names):
    res = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return res.stdout.splitlines() if res.returncode == 0 else names


def census(so: Path) -> dict:
    txt = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True, check=True).stdout
    kernels: dict[str, Counter] = {}
    cur = None
    for line in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        op = m.group(1)
        kernels[cur]["_total"] += 1
        for o in OPS:
            if op == o or op.startswith(o + "."):
                kernels[cur][o] += 1
                if ".2CTA" in op:
                    kernels[cur][o + ".2CTA"] += 1
    names = list(kernels)
    pretty = demangle(names)
    out = {}
    for n, p in zip(names, pretty):
        short = re.sub(r"\(.*", "", p)
        short = re.sub(r"^void ", "", short)
        key = short
        i = 2
        while key in out:
            key = f"{short}#{i}"
            i += 1
        out[key] = {"mangled": n, "demangled": p[:300], **dict(kernels[n])}
    return out


def main():
    so = Path(sys.argv[1]) if len(sys.argv) > 1 else SO
    c = census(so)
    (ROOT / "profiles" / "r02_sass_census.json").write_text(json.dumps(c, indent=1))
    cols = ["UTCHMMA", "UTCIMMA", "UTCCP", "UTMALDG", "UTMASTG", "UTMAREDG", "LDTM", "HMMA", "MUFU.EX2",
            "MUFU.TANH", "MUFU.RCP", "_total"]
    lines = ["# SASS census of libiolm_cuda.so (cuobjdump -sass; `profiles/sass_census.py`)", "",
             "Instruction counts per kernel instantiation (static, not dynamic). `.2CTA` variants are",
             "`cta_group::2` (CTA-pair) forms and are included in the base count.", "",
             "| kernel | " + " | ".join(cols) + " |", "|---|" + "---|" * len(cols)]
    tot = Counter()
    for k, v in sorted(c.items()):
        row = [str(v.get(x, 0)) for x in cols]
        extra = " (2CTA: " + ", ".join(f"{x} {v[x + '.2CTA']}" for x in ("UTCHMMA", "UTCIMMA", "UTCCP")
                                      if v.get(x + ".2CTA")) + ")" if any(
            v.get(x + ".2CTA") for x in ("UTCHMMA", "UTCIMMA", "UTCCP")) else ""
        lines.append(f"| `{k[:90]}`{extra} | " + " | ".join(row) + " |")
        for x in cols:
            tot[x] += v.get(x, 0)
    lines.append("| **total** | " + " | ".join(str(tot[x]) for x in cols) + " |")
    (ROOT / "profiles" / "r02_sass_census.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines[-3:]))


if __name__ == "__main__":
    main()
