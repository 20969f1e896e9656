"""Collect the round-end measurement set (tools/round_measure.sh TAG) from gpurun_out/ into profiles/:
bench lines as r02_bench_*.json, the launch list, ncu --set full summaries (tools/ncu_json.py) and a
markdown table profiles/r02_summary.md.  Usage: python tools/summarize_round.py TAG"""
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r2f"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")
rows = []
for path in sorted(glob.glob(os.path.join(src, f"{tag}_bench_*.json"))):
    name = os.path.basename(path)[len(tag) + 1:]
    try:
        line = [l for l in open(path).read().splitlines() if l.startswith("{")][-1]
        d = json.loads(line)
    except Exception as e:
        print("skip", name, e)
        continue
    shutil.copy(path, os.path.join(dst, "r02_" + name))
    rf = d.get("roofline") or {}
    cfg = d.get("config") or {}
    rows.append((name[:-5], d.get("value"), d.get("unit"), d.get("dtype"), rf.get("us_per_sweep") or rf.get("us_per_batch_sweep"),
                 rf.get("frac"), cfg.get("iters_to_tolerance") or cfg.get("max_iters"),
                 cfg.get("time_to_tolerance_ms"), (d.get("e2e") or {}).get("value"),
                 (d.get("cpu_baseline") or {}).get("value"), (d.get("clocks") or {}).get("sm_mhz")))
for f in glob.glob(os.path.join(src, f"{tag}_launches.csv")):
    shutil.copy(f, os.path.join(dst, "r02_launches_config3.csv"))
ncu = {"res": ("ncu_summary.json", 862, "config 3, 8500-shaped, resident kernel fp64, one solve to tolerance (K = 862)"),
       "batch": ("ncu_summary_config4.json", 20, "config 4, 4096 x 123-shaped scenarios, batch kernel fp64, 20 batch sweeps"),
       "stream": ("ncu_summary_config5.json", 50, "config 5, 64 x 8500 stitched, streaming kernel fp64, 50 sweeps")}
for k, (out, sweeps, wl) in ncu.items():
    rep = os.path.join(src, f"{tag}_{k}.ncu-rep")
    if os.path.exists(rep):
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_json.py"), rep, str(sweeps), wl,
                        os.path.join(dst, out)], check=False)
with open(os.path.join(dst, "r02_summary.md"), "w") as fh:
    fh.write(f"# Round-2 measurement set ({tag}, tools/round_measure.sh; B200, one GPU)\n\n")
    fh.write("| line | value | unit | dtype | us/sweep | roofline frac | K (max) | time to tol. (ms) | e2e | cpu oracle (1 thr) | SM MHz |\n")
    fh.write("|---|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        fh.write("| " + " | ".join("-" if v is None else (f"{v:.4g}" if isinstance(v, float) else str(v)) for v in r) + " |\n")
print(open(os.path.join(dst, "r02_summary.md")).read())
