"""Summarise an ncu launch list (gpu__time_duration per launch) and a --set full capture
into profiles/: a markdown table plus a JSON with the numbers bench.py's roofline cites.

  python tools/ncu_summary.py gpurun_out/launches_r1.csv gpurun_out/prof_r1.ncu-rep profiles/r01
  python tools/ncu_summary.py --capture gpurun_out/sa.ncu-rep profiles/r01_sa "what was captured"
  python tools/ncu_summary.py --bench gpurun_out/launches_cfg3.csv gpurun_out/cfg3.ncu-rep cfg3 65536
"""
import csv
import io
import json
import subprocess
import sys


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = {}, {}
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        k = r[ik].split("(")[0]
        tot[k] = tot.get(k, 0.0) + float(r[iv].replace(",", ""))
        cnt[k] = cnt.get(k, 0) + 1
    s = sum(tot.values())
    return [dict(kernel=k, launches=cnt[k], total_ns=tot[k], avg_us=tot[k] / cnt[k] / 1e3, share=tot[k] / s)
            for k in sorted(tot, key=lambda k: -tot[k])]


WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active": "tmem_pipe_pct",
    "lts__t_sectors_srcunit_tex_lookup_hit.sum": "l2_hit_sectors",
    "lts__t_sectors_srcunit_tex_lookup_miss.sum": "l2_miss_sectors",
    "lts__t_sectors_srcunit_tex.sum.pct_of_peak_sustained_elapsed": "l2_tex_sector_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "gpc__cycles_elapsed.max": "cycles",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed": "smem_pipe_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def full_capture(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for h, u, v in zip(hdr, units, vals):
        if h in WANT:
            x = float(v.replace(",", ""))
            if u in UNITS:
                x *= UNITS[u]
            d[WANT[h]] = x
    return d


def capture_only(rep, prefix, what):
    F = full_capture(rep)
    traffic = F.get("dram_read", 0.0) + F.get("dram_write", 0.0)
    json.dump({"capture": F, "traffic_bytes_per_launch": traffic, "what": what, "source": rep},
              open(prefix + "_ncu.json", "w"), indent=1)
    with open(prefix + "_ncu.md", "w") as f:
        f.write(f"# ncu --set full capture\n\n{what}\n\n| metric | value |\n|---|---|\n")
        for k, v in F.items():
            f.write(f"| {k} | {v:.6g} |\n" if isinstance(v, float) else f"| {k} | {v} |\n")
        f.write(f"| traffic = dram read + write (bytes/launch) | {traffic:.6g} |\n")
    print(json.dumps(F, indent=1))


def bench_capture(launches, rep, name, batch):
    """profiles/r02/<name>_ncu_full.{json,md}: the capture bench.py cites for roofline.traffic
    (its batch, capture date and the commit it was taken at)."""
    import datetime
    import os
    F = full_capture(rep)
    traffic = F.get("dram_read", 0.0) + F.get("dram_write", 0.0)
    commit = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip()
    date = datetime.datetime.fromtimestamp(os.path.getmtime(rep)).strftime("%Y-%m-%d %H:%M")
    L = launch_shares(launches) if launches != "-" else []
    out = {"config": name, "batch": int(batch), "captured": date, "commit": commit, "traffic_bytes_per_launch": traffic,
           "top_kernel_full": F, "launch_list": L, "source": {"launches": launches, "capture": rep}}
    prefix = os.path.join("profiles", "r02", f"{name}_ncu_full")
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu: {name} (B = {batch}), captured {date} at commit {commit}\n\n")
        if L:
            f.write("## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n")
            f.write("| kernel | launches | avg us | share |\n|---|---|---|---|\n")
            for r in L:
                f.write(f"| `{r['kernel']}` | {r['launches']} | {r['avg_us']:.1f} | {r['share']*100:.2f}% |\n")
        f.write("\n## Contraction kernel, --set full\n\n| metric | value |\n|---|---|\n")
        for k, v in F.items():
            f.write(f"| {k} | {v:.6g} |\n" if isinstance(v, float) else f"| {k} | {v} |\n")
        f.write(f"| traffic = dram read + write (bytes/launch) | {traffic:.6g} |\n")
    print(prefix, "traffic", traffic)


def main():
    if sys.argv[1] == "--bench":
        bench_capture(*sys.argv[2:6])
        return
    if sys.argv[1] == "--capture":
        capture_only(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
        return
    launches, rep, prefix = sys.argv[1:4]
    L = launch_shares(launches)
    F = full_capture(rep)
    traffic = F.get("dram_read", 0.0) + F.get("dram_write", 0.0)
    summary = {"launch_list": L, "top_kernel_full": F, "traffic_bytes_per_launch": traffic,
               "source": {"launches": launches, "capture": rep}}
    json.dump(summary, open(prefix + "_ncu.json", "w"), indent=1)
    with open(prefix + "_ncu.md", "w") as f:
        f.write("# ncu summary\n\n## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n")
        f.write("| kernel | launches | avg us | share |\n|---|---|---|---|\n")
        for r in L:
            f.write(f"| `{r['kernel']}` | {r['launches']} | {r['avg_us']:.1f} | {r['share']*100:.2f}% |\n")
        f.write("\n## Top kernel, --set full\n\n| metric | value |\n|---|---|\n")
        for k, v in F.items():
            f.write(f"| {k} | {v:.6g} |\n" if isinstance(v, float) else f"| {k} | {v} |\n")
        f.write(f"| traffic = dram read + write (bytes/launch) | {traffic:.6g} |\n")
    print(json.dumps(summary["top_kernel_full"], indent=1))
    print("traffic", traffic)


if __name__ == "__main__":
    main()
