"""Summarise an ncu --set full report (raw page + source page) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/name.md [--passes N]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def ncu(rep, page):
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                       text=True, check=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def main():
    rep, out = sys.argv[1], sys.argv[2]
    passes = int(sys.argv[sys.argv.index("--passes") + 1]) if "--passes" in sys.argv else None
    raw = ncu(rep, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    lines = [f"# ncu summary: `{rep.split('/')[-1]}`", ""]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    lines.append(f"kernel: `{name}`")
    lines.append("")
    lines.append("| metric | value | unit |")
    lines.append("|---|---|---|")
    got = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"| {k} | {vals[i]} | {units[i]} |")
            got[k] = (vals[i], units[i])
    if passes is None and "--alg-bytes" in sys.argv and "dram__bytes_read.sum" in got:
        # passes of the captured launch: each streams X once (read bytes / bytes of X)
        alg = float(sys.argv[sys.argv.index("--alg-bytes") + 1])
        v, u = got["dram__bytes_read.sum"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        passes = max(1, round(float(v.replace(",", "")) * scale / alg))
    if passes and "dram__bytes_read.sum" in got:
        v, u = got["dram__bytes_read.sum"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        w, uw = got.get("dram__bytes_write.sum", ("0", "byte"))
        sw = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(uw, 1)
        tot = float(v.replace(",", "")) * scale + float(w.replace(",", "")) * sw
        lines.append("")
        lines.append(f"DRAM traffic per streaming pass ({passes} passes in the launch): "
                     f"{tot / passes / 1e6:.1f} MB")
        if "--traffic-json" in sys.argv:   # read by bench.py (roofline.traffic)
            import json
            with open(sys.argv[sys.argv.index("--traffic-json") + 1], "w") as fh:
                json.dump({"dram_bytes_per_pass": tot / passes, "report": rep.split("/")[-1],
                           "passes_in_launch": passes}, fh)
    # stall reasons
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(vals[i].replace(",", "")), h.replace(
                    "smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    lines += ["", "## warp-state samples (all)", "", "| reason | share |", "|---|---|"]
    for s, h in sorted(stalls, reverse=True)[:10]:
        lines.append(f"| {h} | {100 * s / tot:.1f}% |")
    # source page: opcode mix and stall by opcode
    src = ncu(rep, "source")
    h2 = src[1]
    try:
        iS, iE, iSrc = (h2.index("Warp Stall Sampling (All Samples)"),
                        h2.index("Instructions Executed"), h2.index("Source"))
        cs, ce = Counter(), Counter()
        for r in src[2:]:
            try:
                s, e = float(r[iS] or 0), float(r[iE] or 0)
            except (ValueError, IndexError):
                continue
            op = r[iSrc].split()
            if not op:
                continue
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            o = o.split(".")[0]
            cs[o] += s
            ce[o] += e
        ts, te = sum(cs.values()) or 1, sum(ce.values()) or 1
        lines += ["", "## SASS opcodes (stall samples / executed)", "",
                  "| opcode | stall share | instr share |", "|---|---|---|"]
        for o, s in cs.most_common(14):
            lines.append(f"| {o} | {100 * s / ts:.1f}% | {100 * ce[o] / te:.1f}% |")
        tma = [o for o in ce if o.startswith("UBLKCP") or o.startswith("UTMA")]
        lines.append("")
        lines.append(f"bulk-copy / TMA opcodes present: {', '.join(sorted(tma)) or 'none'}")
    except ValueError:
        pass
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
