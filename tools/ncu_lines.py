"""Per-source-line instruction / stall-sample shares of one kernel in an ncu
report (--set full --import-source on): where the issue slots go.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, timeout=600).stdout
    cur, hdr, res = None, None, []
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "Function Name" or not r[0] or not hdr:
            continue
        try:
            ie, ti, samp = int(r[7]), int(r[8]), int(r[4])
        except ValueError:
            continue
        res.append((ie, ti, samp, cur, r[0], r[1][:90]))
    tot = sum(x[0] for x in res) or 1
    tots = sum(x[2] for x in res) or 1
    print(f"total warp instructions {tot}, stall samples {tots}")
    for x in sorted(res, reverse=True)[:top]:
        print(f"{x[0] / tot * 100:5.1f}% inst {x[2] / tots * 100:5.1f}% samples "
              f"{x[1] / max(x[0], 1):4.1f} thr/inst  {x[3]}:{x[4]}  {x[5]}")


if __name__ == "__main__":
    main()
