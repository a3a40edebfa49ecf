"""Copy a gpurun evidence run (scripts/evidence.sh -> gpurun_out/) into
profiles/<tag>_* and move an older tag's top-level files under profiles/<dir>/.

    python scripts/store_evidence.py r02i [--archive r02f --into r02_history]
"""
import glob
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def main():
    tag = sys.argv[1]
    if "--archive" in sys.argv:
        old = sys.argv[sys.argv.index("--archive") + 1]
        into = sys.argv[sys.argv.index("--into") + 1] if "--into" in sys.argv else old
        os.makedirs(os.path.join(PROF, into), exist_ok=True)
        for f in glob.glob(os.path.join(PROF, f"{old}_*")):
            if "sanitizer" in f:  # the last sanitizer logs stay on top
                continue
            shutil.move(f, os.path.join(PROF, into, os.path.basename(f)))
    copied = []
    for f in glob.glob(os.path.join(OUT, "bench_*.json")):
        dst = os.path.join(PROF, f"{tag}_" + os.path.basename(f))
        shutil.copy(f, dst)
        copied.append(dst)
    for f in glob.glob(os.path.join(OUT, f"{tag}_*")):
        if f.endswith((".log", ".err", ".ncu-rep")) or f.endswith("incontext.csv"):
            continue
        shutil.copy(f, os.path.join(PROF, os.path.basename(f)))
        copied.append(f)
    for name in ("pytest_gpu.log", "smoke.log", "ingest.json"):
        src = os.path.join(OUT, name)
        if os.path.exists(src):
            shutil.copy(src, os.path.join(PROF, f"{tag}_{name}"))
            copied.append(src)
    print(f"{len(copied)} files -> profiles/{tag}_*")


if __name__ == "__main__":
    main()
