"""Per-source-line hot spots of one kernel in an ncu report (cuda,sass view): stall samples and
executed warp instructions aggregated by (file, line)."""
import csv
import subprocess
import sys


def main(rep, kernel, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kernel}"], capture_output=True, text=True).stdout
    agg = {}
    f = "?"
    cur = None
    tot_s = tot_i = 0
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0]:
            cur = (f, int(r[0]), r[1][:90])
            try:
                s, i = float(r[4]), float(r[7])
            except ValueError:
                continue
            a = agg.setdefault(cur, [0, 0])
            a[0] += s
            a[1] += i
            tot_s += s
            tot_i += i
    rows = sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]
    print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3g}")
    for (fn, ln, src), (s, i) in rows:
        print(f"{100 * s / tot_s:5.1f}% samp {100 * i / tot_i:5.1f}% inst  {fn}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
