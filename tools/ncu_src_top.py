"""Top source lines by warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`.

    python tools/ncu_src_top.py report.ncu-rep [N] [file-substring]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    filt = sys.argv[3] if len(sys.argv) > 3 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, rows = None, None, []
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] in ("", "Function Name"):
            continue
        d = dict(zip(hdr, rec))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
        except (ValueError, KeyError):
            continue
        if s == 0:
            continue
        stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
        rows.append((s, fname.split("/")[-1], int(rec[0]), rec[1].strip()[:70], stalls, d.get("Instructions Executed", "")))
    tot = sum(r[0] for r in rows)
    print(f"total samples {tot}")
    for s, f, ln, src, st, ie in sorted(rows, reverse=True)[:top]:
        if filt and filt not in f:
            continue
        top3 = " ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:4])
        print(f"{100*s/tot:5.1f}% {f}:{ln:<4} inst={ie:>8} | {top3} | {src}")


if __name__ == "__main__":
    main()
