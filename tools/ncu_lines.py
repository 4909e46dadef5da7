"""Per-source-line instruction and stall-sample shares of an ncu --import-source report.

    python tools/ncu_lines.py report.ncu-rep [--top 40]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr, agg = None, None, {}
    for r in rows:
        if len(r) == 2 and r[0] in ("File Path", "Function Name"):
            if r[0] == "File Path":
                cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 8 or r[0] == "":
            continue
        ie = int(r[7]) if r[7].isdigit() else 0
        sm = int(r[6]) if r[6].isdigit() else 0
        key = (cur, int(r[0]), r[1].strip()[:90])
        a, b = agg.get(key, (0, 0))
        agg[key] = (a + ie, b + sm)
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"warp instructions {ti}, stall samples {ts}")
    print("| inst % | samples % | line | source |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"| {v[0] / ti * 100:.1f} | {v[1] / ts * 100:.1f} | {k[0]}:{k[1]} | `{k[2]}` |")


if __name__ == "__main__":
    main()
