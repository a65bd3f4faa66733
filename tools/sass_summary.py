"""Static per-kernel SASS summary of the library: registers/smem (cuobjdump -res-usage),
instruction count and the mnemonics that evidence the design (MUFU, ATOMS, REDG, VOTE...)."""
import collections
import re
import subprocess
import sys

KEY = ("MUFU.EX2", "MUFU.RSQ", "MUFU.RCP", "ATOMS", "REDG", "ATOMG", "VOTE", "SHFL", "BAR.SYNC", "LDS", "STS", "FFMA2",
       "DFMA", "DADD", "DMUL", "FFMA", "LDG", "STG", "UTMALDG", "UTCHMMA", "HMMA")


def main(so):
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", so], capture_output=True, text=True).stdout
    usage = {}
    fn = None
    for ln in res.splitlines():
        m = re.search(r"Function (\S+):", ln)
        if m:
            fn = m.group(1)
        m = re.search(r"REG:(\d+).*SHARED:(\d+)", ln)
        if m and fn:
            usage[fn] = (int(m.group(1)), int(m.group(2)))
    counts, total, fn = {}, collections.Counter(), None
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if m and fn:
            op = m.group(1)
            counts[fn]["_total"] += 1
            for k in KEY:
                if op.startswith(k):
                    counts[fn][k] += 1
    demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
    for (fn, c), name in zip(counts.items(), demangle):
        reg, smem = usage.get(fn, (0, 0))
        keys = ", ".join(f"{k} {c[k]}" for k in KEY if c[k])
        print(f"{name[:70]:70s} regs {reg:3d} smem {smem:6d} B  instr {c['_total']:6d}  | {keys}")


if __name__ == "__main__":
    main(sys.argv[1])
