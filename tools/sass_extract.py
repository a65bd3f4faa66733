"""Extract one kernel's SASS from `cuobjdump -sass <so>` (tools for profiles/)."""
import subprocess
import sys


def extract(so, fn):
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    keep, lines = False, []
    for ln in out.splitlines():
        if "Function :" in ln:
            keep = ln.strip().endswith(fn)
        if keep:
            lines.append(ln)
    return "\n".join(lines)


if __name__ == "__main__":
    print(extract(sys.argv[1], sys.argv[2]))
