"""Summarise the first kernel of an ncu --set full report as the JSON bench.py reads for `traffic`:
python tools/ncu_json.py REPORT.ncu-rep SWEEPS_PER_LAUNCH "workload text" OUT.json"""
import csv
import json
import subprocess
import sys

rep, sweeps, workload, out = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h, u, v = rows[0], rows[1], rows[2]


def g(k, scale=1.0):
    i = h.index(k)
    x = float(v[i].replace(",", ""))
    unit = u[i]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
            "second": 1, "%": 1, "": 1, "register/thread": 1}.get(unit, 1)
    return x * mult * scale


dur = g("gpu__time_duration.sum")
rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
d = {"report": rep.split("/")[-1], "kernel": v[h.index("Kernel Name")], "duration_s": dur,
     "dram_bytes_read": rd, "dram_bytes_write": wr, "sweeps_per_launch": sweeps,
     "lts_hit_pct": g("lts__t_sector_hit_rate.pct"), "l1_hit_pct": g("l1tex__t_sector_hit_rate.pct"),
     "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
     "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
     "registers": g("launch__registers_per_thread"), "workload": workload,
     "dram_bytes_per_sweep": (rd + wr) / sweeps, "us_per_sweep_under_ncu": dur * 1e6 / sweeps,
     "dram_gbs": (rd + wr) / dur / 1e9}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d))
