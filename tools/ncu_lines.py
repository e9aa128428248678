"""Top CUDA source lines by warp-stall samples from an ncu report (needs -lineinfo)."""
import csv
import subprocess
import sys


def main(rep, skip, top=25, by="stall"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(skip), "--launch-count",
                          "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, lines = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0]:
            d = dict(zip(hdr[4:], r[4:]))
            try:
                lines.append((float(d.get("Warp Stall Sampling (All Samples)", 0) or 0),
                              float(d.get("Instructions Executed", 0) or 0), cur, r[0], r[1].strip()))
            except ValueError:
                pass
    tot = sum(x[0] for x in lines) or 1
    toti = sum(x[1] for x in lines) or 1
    print(f"samples {tot:.0f}  instructions {toti:.3g}")
    key = (lambda x: -x[1]) if by == "inst" else (lambda x: -x[0])
    for s, i, f, ln, src in sorted(lines, key=key)[:top]:
        print(f"{100 * s / tot:5.1f}% stall {100 * i / toti:5.1f}% inst  {f}:{ln}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 25,
         sys.argv[4] if len(sys.argv) > 4 else "stall")
