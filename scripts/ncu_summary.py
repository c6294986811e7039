"""Summarise ncu reports (gpurun_out/tma_so*.ncu-rep) into profiles/ncu_summary.json + a text table."""
import csv, io, json, subprocess, sys, os
from collections import OrderedDict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
           "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "launch__registers_per_thread",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__block_size", "smsp__cycles_active.avg"]

def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}

def num(v):
    try: return float(v.replace(",", ""))
    except Exception: return None

def main(tag, files, pts, key="k_tma", steps=1, summ=None, lines=None):
    summ = summ or {"tag": tag}
    summ[key] = OrderedDict()
    lines = lines if lines is not None else [f"# ncu --set full --clock-control none, 256^3, {tag}", ""]
    lines.append(f"## {key}: one launch = {steps} time step(s)")
    for so, path in files:
        d = raw(path)
        e = OrderedDict()
        for m in METRICS:
            if m in d: e[m] = [num(d[m][0]), d[m][1]]
        def to_bytes(x):
            v, u = x; f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1); return v * f
        rd, wr = to_bytes(e["dram__bytes_read.sum"]), to_bytes(e["dram__bytes_write.sum"])
        dur = e["gpu__time_duration.sum"][0] * {"usecond": 1e-6, "us": 1e-6, "nsecond": 1e-9, "ns": 1e-9, "msecond": 1e-3, "ms": 1e-3}[e["gpu__time_duration.sum"][1]]
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v[0]) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and num(v[0])}
        p = pts[so] * steps  # point updates per launch
        e["steps_per_launch"] = steps
        e["dram_bytes_per_launch"] = rd + wr
        e["dram_bytes_per_point"] = (rd + wr) / p
        e["algorithmic_bytes_per_point"] = 20
        e["duration_s"] = dur
        e["gpts"] = p / dur / 1e9
        e["stall_samples"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
        summ[key][f"so{so}"] = e
        lines.append(f"SO {so}: {dur*1e6:.1f} us  {p/dur/1e9:.1f} GPts/s  DRAM read {rd/1e6:.1f} MB write {wr/1e6:.1f} MB "
                     f"({(rd+wr)/p:.2f} B/pt vs 20 algorithmic)  DRAM {e['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'][0]:.1f}% "
                     f"L2 hit {e['lts__t_sector_hit_rate.pct'][0]:.1f}%  issue {e['smsp__issue_active.avg.pct_of_peak_sustained_active'][0]:.1f}%  "
                     f"regs {e['launch__registers_per_thread'][0]:.0f}  smem conflicts {e['l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum'][0]:.0f}/"
                     f"{e['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'][0]:.0f} wavefronts")
        lines.append("   top stalls: " + ", ".join(f"{k} {v:.0f}" for k, v in list(e["stall_samples"].items())[:6]))
    lines.append("")
    return summ, lines

if __name__ == "__main__":
    tag = sys.argv[1]
    files = []
    for so in (4, 8, 12, 16):
        p = f"gpurun_out/tma_so{so}.ncu-rep"
        if os.path.exists(p): files.append((so, p))
    pts = {so: (256 - so) ** 3 for so in (4, 8, 12, 16)}
    summ, lines = main(tag, files, pts)
    tb = [(so, f"gpurun_out/tb_so{so}.ncu-rep") for so in (4, 8, 12, 16) if os.path.exists(f"gpurun_out/tb_so{so}.ncu-rep")]
    if tb:
        summ, lines = main(tag, tb, pts, key="k_tma_tb", steps=2, summ=summ, lines=lines)
    text = "\n".join(lines) + "\n"
    # merge: keep the other captures' keys (steady-state ranges, retired-kernel history)
    old = json.load(open("profiles/ncu_summary.json")) if os.path.exists("profiles/ncu_summary.json") else {}
    if "k_tma" in old and old.get("tag") != tag:
        old[f"k_tma_{old.get('tag', 'prev')}"] = old["k_tma"]
    old.update(summ)
    json.dump(old, open("profiles/ncu_summary.json", "w"), indent=1)
    open(f"profiles/ncu_k_tma_{tag}.txt", "w").write(text)
    print(text)
