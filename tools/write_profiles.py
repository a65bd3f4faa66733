"""Regenerate profiles/ from the ncu outputs of tools/capture_profiles.sh.

    python tools/write_profiles.py [--tag r01]

Reads gpurun_out/launches.csv (launch list of a bench run), gpurun_out/cycle_cfg3.ncu-rep
(--set full of K1/K2/K3 of one cfg3 cycle) and gpurun_out/k2_cfg3.ncu-rep (--set full of
K2 alone, source-level) and writes:
  profiles/<tag>_launches_cfg3.csv, <tag>_launch_shares.txt, <tag>_ncu_cycle_cfg3.txt,
  profiles/ncu_summary.json (the K2 figures bench.py quotes in its roofline block),
  <tag>_ncu_k2_reference_mode.txt, <tag>_ncu_frows.txt and the SASS listings / summary of
  the in-tree library (cuobjdump, here).
"""
import argparse
import collections
import contextlib
import csv
import io
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)

import ncu_lines  # noqa: E402
import ncu_opmix  # noqa: E402
import ncu_summary  # noqa: E402

PSTEPS = 8 * 262144 * 250


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        tot[r[4]] += float(r[14])
        cnt[r[4]] += 1
    s = sum(tot.values()) or 1.0
    out = []
    for k, v in tot.most_common():
        out.append((k, cnt[k], v / 1e6, 100 * v / s))
    return out


def capture(fn, *a):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        fn(*a)
    return buf.getvalue()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--prof-dir", default=None, help="write here instead of profiles/ (e.g. on the GPU box)")
    a = ap.parse_args()
    prof = a.prof_dir or os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    src = os.path.join(ROOT, a.out)

    shares = launch_shares(os.path.join(src, "launches.csv"))
    shutil.copy(os.path.join(src, "launches.csv"), os.path.join(prof, f"{a.tag}_launches_cfg3.csv"))
    with open(os.path.join(prof, f"{a.tag}_launch_shares.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 3 "
                "--warmup 3 --no-cpu-baseline --no-ref-mode --lat-cycles 0\n# (the bench's device cycles + its "
                "chunked e2e cycles; cold-cache, serialised launches: compare shares, not absolutes)\n")
        for k, n, ms, pct in shares:
            f.write(f"{k[:60]:60s} n={n:4d} total={ms:9.3f} ms share={pct:5.1f}%\n")
    k2_share = next((p for k, n, ms, p in shares if "k_predict" in k), None)

    cyc = os.path.join(src, "cycle_cfg3.ncu-rep")
    k2 = os.path.join(src, "k2_cfg3.ncu-rep")
    text = ["# ncu --set full --clock-control none of one update+predict cycle (cfg3: 8 humans x 262144 "
            "particles x 250 steps, 400x400)",
            "# command: tools/capture_profiles.sh; B200, driver 580, CUDA 12.9, sm_100a; per-launch values"]
    text.append(capture(ncu_summary.main, cyc))
    mix = capture(ncu_opmix.main, k2, PSTEPS)
    text.append("# k_predict dynamic SASS opcode mix (lane-instructions per particle-step)\n" + mix)
    text.append("# k_predict per-source-line warp-stall samples\n" + capture(ncu_lines.main, k2, 40))
    open(os.path.join(prof, f"{a.tag}_ncu_cycle_cfg3.txt"), "w").write("\n".join(text))

    SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
             "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3}
    recs, units = ncu_summary.load(k2)
    d = recs[0]

    def f(k, rec=None, unit_map=None):
        """value in base units: bytes, milliseconds, or as reported"""
        r, u = (rec or d), (unit_map or units)
        return float(r[k].replace(",", "")) * SCALE.get(u.get(k, ""), 1.0)
    ipp = f("smsp__inst_executed.sum") * 32 / PSTEPS
    mufu = 0.0
    for ln in mix.splitlines():
        if ln.strip().startswith("MUFU"):
            mufu = float(ln.split("per-pstep")[1].split()[0])
    cyc_recs, cyc_units = ncu_summary.load(cyc)
    by = {r.get("Kernel Name", ""): r for r in cyc_recs}
    get = lambda name, k: next((round(f(k, r, cyc_units), 4) for n, r in by.items() if name in n and k in r), None)  # noqa: E731
    dram = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
    summary = {"production": {
        "k_predict": {
            "source": f"profiles/{a.tag}_ncu_cycle_cfg3.txt (ncu --set full, cfg3: 8 humans x 262144 particles x 250 steps)",
            "duration_ms": round(f("gpu__time_duration.sum"), 3),
            "issue_active_pct": round(f("smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
            "lane_instr_per_particle_step": round(ipp, 1),
            "mufu_per_particle_step": round(mufu, 1),
            "dram_bytes_per_launch": int(dram),
            "registers_per_thread": int(f("launch__registers_per_thread")),
            "xu_pipe_pct": round(f("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"), 1),
            "share_of_cycle_pct": round(k2_share, 1) if k2_share else None,
        },
        "k_epilogue": {"duration_ms": get("k_epilogue", "gpu__time_duration.sum"),
                       "issue_active_pct": get("k_epilogue", "smsp__issue_active.avg.pct_of_peak_sustained_active")},
        "k_belief": {"duration_ms": get("k_belief", "gpu__time_duration.sum")},
    }}
    json.dump(summary, open(os.path.join(prof, "ncu_summary.json"), "w"), indent=2)
    print(json.dumps(summary, indent=1))

    # reference-arithmetic K2 and the f-row kernels
    ref = os.path.join(src, "k2_refmode.ncu-rep")
    if os.path.exists(ref):
        open(os.path.join(prof, f"{a.tag}_ncu_k2_reference_mode.txt"), "w").write(
            "# ncu --set full of the REFERENCE-arithmetic kernel k_predict<0,4,0,0> at the cfg3 launch shape (8 humans x "
            "262144 particles x 20 steps, K = 4 particles per thread)\n" + capture(ncu_summary.main, ref) + "\n# dynamic SASS opcode mix (lane-instructions per "
            "particle-step)\n" + capture(ncu_opmix.main, ref, 8 * 262144 * 20))
    ext = os.path.join(src, "extras.ncu-rep")
    if os.path.exists(ext):
        open(os.path.join(prof, f"{a.tag}_ncu_frows.txt"), "w").write(
            "# ncu --set full of the f-row kernels (tools/profile_extras.py): collision field of a 250x400x400 f32 "
            "union,\n# MPPI 4096 rollouts x 40 steps against that mask, exact enumeration 100x100 cells x 96 actions "
            "x 10 hyps\n# (tools/capture_profiles.sh; per-launch values)\n" + capture(ncu_summary.main, ext))
    aux = os.path.join(src, "aux.ncu-rep")
    if os.path.exists(aux):
        open(os.path.join(prof, f"{a.tag}_ncu_aux_kernels.txt"), "w").write(
            "# ncu --set full of the remaining kernels (ordered unions, time union, predict_naive, emplace, "
            "smooth,\n# sample_hypotheses, propagate_step) at tools/sanitize_run.py's small sizes: latency-bound "
            "utility launches,\n# listed for completeness (tools/capture_profiles.sh; per-launch values)\n"
            + capture(ncu_summary.main, aux))
    pub = os.path.join(src, "publish.ncu-rep")
    if os.path.exists(pub):
        open(os.path.join(prof, f"{a.tag}_ncu_publish.txt"), "w").write(
            "# ncu --set full of k_publish (tile-sparse D2H of the f64 fused union into the pinned host stack, "
            "one launch per horizon chunk of the e2e cycle; kernel stores over PCIe)\n"
            "# (tools/capture_profiles.sh; per-launch values)\n" + capture(ncu_summary.main, pub))
    # SASS of the cycle kernels and the static summary of every kernel in the library
    import sass_extract
    import sass_summary
    so = os.path.join(ROOT, "paper_2603_01122_b200", "_lib", "libgridcast_b200.so")
    for name, fn in (("k_predict_production", "_ZN2gc9k_predictILi4ELi4ELb0ELb0EEEvNS_7KParamsE"),
                     ("k_epilogue", "_ZN2gc12k_epilogue_rILi3EEEvNS_7EParamsE"),
                     ("k_belief", "_ZN2gc8k_beliefILi8EEEvNS_7BParamsE")):
        open(os.path.join(prof, f"{a.tag}_sass_{name}.txt"), "w").write(sass_extract.extract(so, fn) + "\n")
    open(os.path.join(prof, f"{a.tag}_sass_summary_all_kernels.txt"), "w").write(capture(sass_summary.main, so))


if __name__ == "__main__":
    main()
