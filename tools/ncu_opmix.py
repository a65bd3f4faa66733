"""Dynamic SASS opcode mix of an ncu report (source page), per particle-step."""
import collections
import csv
import io
import subprocess
import sys


def main(path, psteps):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    I, S, W = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    ops, stall, tot = collections.Counter(), collections.Counter(), 0
    for r in rows[2:]:
        if len(r) <= I or not r[S].strip():
            continue
        try:
            n = int(r[I] or 0)
        except ValueError:
            continue
        tok = r[S].strip().split()
        op = tok[1] if tok[0].startswith("@") else tok[0]
        ops[op.split(".")[0]] += n
        stall[op.split(".")[0]] += int(r[W] or 0)
        tot += n
    print(f"warp-instr {tot}, lane-instr per particle-step {tot * 32 / psteps:.1f}")
    for op, n in ops.most_common(24):
        print(f"  {op:10s} {100 * n / tot:5.1f}%  per-pstep {n * 32 / psteps:7.1f}  stall-samples {stall[op]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
