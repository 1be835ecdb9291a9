"""Per kernel-class statistics from an ncu launch list (never a bench number).

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -s 3000 -c 400 --csv --log-file gpurun_out/<cfg>_launches.csv python profiles/profile_run.py ...
  python profiles/launch_stats.py gpurun_out/<cfg>_launches.csv <cfg>   # -> profiles/traffic.json[<cfg>]

Classes follow the engine's per-layer launch order: QKV GEMM, prefill attention, decode attention,
[quant], Wo GEMM (first residual GEMM after attention), LN, W_in GEMM, [quant], W_out GEMM, LN.
ncu serialises launches and runs them cold, so shares (not absolute times) are what compare with
bench.py's live CUDA-event timings."""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path


def classify(name: str, state: dict) -> str:
    if "attn_prefill" in name:
        state["after_attn"] = True
        return "attn_prefill"
    if "attn_decode" in name:
        state["after_attn"] = True
        return "attn_decode"
    if "embed_ln" in name:
        return "embed_ln"
    if "ln_" in name:
        return "ln"
    if "quant_rows" in name:
        return "quant"
    if "head_argmax" in name:
        return "head"
    if "gemm" in name:
        # template args: gemm_tn_kernel<BN, EPI, ...> / gemm_sp_kernel<EPI>
        args = name.split("<", 1)[1].split(">", 1)[0]
        parts = [p.strip(" ()int") for p in args.split(",")]
        epi = int(parts[0] if "gemm_sp" in name else parts[1])
        if epi == 4:
            return "gemm_qkv"
        if epi == 2:
            return "gemm_in"
        if epi == 3:
            if state.pop("after_attn", False):
                return "gemm_o"
            return "gemm_out"
    return "other"


def main(path: str, cfg: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr_i]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        try:
            per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        names[r[ii]] = r[ki]
    state, agg = {}, defaultdict(lambda: [0, 0.0, 0.0])
    for lid in sorted(per, key=int):
        c = classify(names[lid], state)
        m = per[lid]
        a = agg[c]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'class':14s} {'launches':>8s} {'share':>7s} {'avg us':>9s} {'DRAM MB/launch':>15s}")
    out = {}
    for c, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{c:14s} {n:8d} {100 * t / tot:6.1f}% {t / n / 1e3:9.1f} {b / n / 1e6:15.1f}")
        out[c] = int(b / n)
    prof = Path(__file__).resolve().parent / "traffic.json"
    data = json.loads(prof.read_text()) if prof.exists() else {}
    data = {k: v for k, v in data.items() if isinstance(v, dict) or k == "_source"}
    data["_source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (profiles/launch_stats.py): mean "
                       "DRAM bytes per launch of each kernel class in the bench's steady state, per config")
    data[cfg] = out
    prof.write_text(json.dumps(data, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
