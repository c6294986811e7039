"""Summarise the steady-state ncu captures (scripts/ncu_steady.sh -> gpurun_out/ncu_steady_*.csv)
into profiles/ncu_summary.json["k_tma_steady"] and copy the CSVs to profiles/ (tagged)."""
import csv
import glob
import io
import json
import os
import shutil
import statistics
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
summ_path = "profiles/ncu_summary.json"
summ = json.load(open(summ_path))
out = summ.setdefault("k_tma_steady", {})
for f in sorted(glob.glob("gpurun_out/ncu_steady_*.csv")):
    name = os.path.basename(f)[len("ncu_steady_"):-4]  # e.g. 8_256, 8_512_damp, persist_8_256
    parts = name.split("_")
    if not parts[0].isdigit():
        continue
    so, n = int(parts[0]), int(parts[1])
    damp = len(parts) > 2 and parts[2] == "damp"
    txt = open(f).read()
    i = txt.find('"ID"')
    if i < 0:
        continue
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    by = {}
    for r in rows:
        by.setdefault(r["Metric Name"], []).append(float(r["Metric Value"].replace(",", "")))
    rd, wr = statistics.mean(by["dram__bytes_read.sum"]), statistics.mean(by["dram__bytes_write.sum"])
    t = statistics.mean(by["gpu__time_duration.sum"]) * 1e-9
    pts = (n - so) ** 3
    key = f"n{n}_so{so}" + ("_damp" if damp else "")
    out[key] = {"launches": len(by["dram__bytes_read.sum"]), "dram_bytes_per_launch": rd + wr,
                "dram_read_bytes_per_point": round(rd / pts, 3), "dram_write_bytes_per_point": round(wr / pts, 3),
                "dram_bytes_per_point": round((rd + wr) / pts, 3), "launch_ns_under_ncu": round(t * 1e9),
                "dram_gbs_under_ncu": round((rd + wr) / t / 1e9, 1), "dram_frac_under_ncu": round((rd + wr) / t / 1e9 / peak, 4),
                "source": f"profiles/ncu_steady_{tag}_{name}.csv"}
    shutil.copy(f, f"profiles/ncu_steady_{tag}_{name}.csv")
summ["k_tma_steady_note"] = ("launches 31..42 of a 50-step run under ncu --cache-control none --clock-control "
                             "none (scripts/ncu_steady.sh): every launch sees the L2 state its predecessor left; "
                             "ncu serialises launches (no PDL overlap), so times are per launch, not per step")
json.dump(summ, open(summ_path, "w"), indent=1)
print(json.dumps(out, indent=1))
