"""Per-source-line hot spots of one kernel in an ncu report (--import-source on).

    python tools/ncu_lines.py report.ncu-rep [top]
Aggregates the `--page source --print-source=cuda,sass` CSV by CUDA line:
stall samples and executed warp instructions."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, out = None, None, []
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if not r[0].isdigit() or hdr is None:
            continue
        try:
            samp = int(r[4])
            ins = int(r[7])
        except (ValueError, IndexError):
            continue
        out.append((samp, ins, cur, int(r[0]), r[1][:100]))
    tot = sum(o[0] for o in out) or 1
    toti = sum(o[1] for o in out) or 1
    print(f"stall samples {tot}  warp instructions {toti}")
    for o in sorted(out, reverse=True)[:top]:
        print(f"{100 * o[0] / tot:5.1f}% {100 * o[1] / toti:5.1f}%  {o[2]}:{o[3]}  {o[4]}")


if __name__ == "__main__":
    main()
