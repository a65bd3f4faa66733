"""Per-CUDA-source-line stall samples and executed instructions of an ncu report."""
import collections
import csv
import io
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname = ""
    agg = collections.defaultdict(lambda: [0, 0, ""])
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        try:
            w = int(r[4] or 0)
            n = int(r[7] or 0)
        except ValueError:
            continue
        key = (fname, line)
        agg[key][0] += w
        agg[key][1] += n
        if not agg[key][2]:
            agg[key][2] = r[1][:100]
    tw = sum(v[0] for v in agg.values()) or 1
    tn = sum(v[1] for v in agg.values()) or 1
    for (f, l), (w, n, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100 * w / tw:5.1f}% stall {100 * n / tn:5.1f}% inst  {f}:{l:<4} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
