"""Copy a gpurun evidence run (scripts/evidence.sh -> gpurun_out/ev_*) into
profiles/<tag>_* and archive the previous top-level tag under profiles/<old>/.

    python scripts/store_evidence.py r01g [--archive r01f]
"""
import csv
import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def main():
    tag = sys.argv[1]
    if "--archive" in sys.argv:
        old = sys.argv[sys.argv.index("--archive") + 1]
        os.makedirs(os.path.join(PROF, old), exist_ok=True)
        for f in glob.glob(os.path.join(PROF, f"{old}_*")):
            shutil.move(f, os.path.join(PROF, old, os.path.basename(f)))
    for f in glob.glob(os.path.join(OUT, "ev_bench_*.json")):
        shutil.copy(f, os.path.join(PROF, f"{tag}_" + os.path.basename(f)[3:]))
    shutil.copy(os.path.join(OUT, "ev_launches.csv"), os.path.join(PROF, f"{tag}_launches.csv"))
    with open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w") as fh:
        fh.write("VATE_PROFILE_REGION=1 ncu --metrics gpu__time_duration.sum --clock-control none "
                 "--profile-from-start off --csv python bench.py --steps 10 --warmup 3\n"
                 "Exactly the 10 timed value-region slices of the default bench (cfg 2: c=24, "
                 "k=60, g=1024, 5M packets, 1M hosts; pipelined slice step, advance fused into "
                 "the bitmap pass).\n")
        fh.write(open(os.path.join(OUT, "ev_launches_summary.txt")).read())
    with open(os.path.join(PROF, f"{tag}_ncu_kernels.txt"), "w") as fh:
        fh.write("# ncu --set full --clock-control none, one steady-state launch each "
                 "(scripts/evidence.sh); cfg 2 unless the report name says cfg4; _full = g0 "
                 "recomputed every slice (--incremental off)\n")
        fh.write(open(os.path.join(OUT, "ev_ncu_kernels.txt")).read())
    for name in ("pytest_gpu.log", "smoke.log"):
        shutil.copy(os.path.join(OUT, "ev_" + name), os.path.join(PROF, f"{tag}_{name}"))
    for t in ("memcheck", "racecheck", "synccheck"):
        f = os.path.join(OUT, f"sanitize_{t}.log")
        if os.path.exists(f):
            shutil.copy(f, os.path.join(PROF, f"{tag}_sanitizer_{t}.log"))
    rep = os.path.join(OUT, "ev_prof_k_scan_packed16.ncu-rep")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) > 2:
        h = rows[1]
        isrc, iw, ie = (h.index("Source"), h.index("Warp Stall Sampling (All Samples)"),
                        h.index("Instructions Executed"))
        data = []
        for r in rows[2:]:
            if len(r) >= len(h):
                data.append((int(r[iw] or 0), r[isrc][:90], r[ie]))
        tot = sum(d[0] for d in data) or 1
        with open(os.path.join(PROF, f"{tag}_scan_source_hotspots.txt"), "w") as fh:
            fh.write("# cfg 2 scan kernel, ncu --set full source page (SASS), warp-stall samples "
                     "per instruction (top 20)\n# " + rows[0][1][:150] + "\n")
            fh.write(f"total samples {tot}\n")
            for d in sorted(data, reverse=True)[:20]:
                fh.write(f"{d[0]:6d} {100 * d[0] / tot:5.1f}%  {d[1]:90s} exec={d[2]}\n")
    print("stored", tag)


if __name__ == "__main__":
    main()
