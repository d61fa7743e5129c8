"""Summarise an ncu --set full report + launch list into profiles/ (JSON + markdown)."""
import csv, io, json, subprocess, sys

rep, launches, out_prefix = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "lts__t_sectors.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "lts__t_sectors_srcunit_ltcfabric.sum", "lts__t_sectors_lookup_hit.sum", "lts__t_sectors_lookup_miss.sum",
        "lts__t_requests_srcunit_tex_op_read.sum", "lts__t_requests_srcunit_tex_op_write.sum",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
d = {}
for k in want:
    for i, h in enumerate(hdr):
        if h == k:
            d[k] = {"value": vals[i], "unit": units[i]}
def num(k, scale=1.0):
    v = d.get(k, {}).get("value")
    try:
        return float(v.replace(",", "")) * scale
    except Exception:
        return None
unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def bytes_of(k):
    u = d.get(k, {}).get("unit", "byte")
    v = num(k)
    return None if v is None else v * unit_scale.get(u, 1)
dram = None
if bytes_of("dram__bytes_read.sum") is not None and bytes_of("dram__bytes_write.sum") is not None:
    dram = bytes_of("dram__bytes_read.sum") + bytes_of("dram__bytes_write.sum")
# launch list
lr = list(csv.reader(open(launches)))
hi = next(i for i, r in enumerate(lr) if "Kernel Name" in r)
h = lr[hi]; ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ls = [(r[ki].split("(")[0], float(r[vi])) for r in lr[hi + 1:] if r[mi] == "gpu__time_duration.sum"]
tot = sum(v for _, v in ls)
agg = {}
for k, v in ls:
    agg.setdefault(k, []).append(v)
l2 = num("lts__t_sectors.sum")
l2r = num("lts__t_sectors_srcunit_tex_op_read.sum")
l2w = num("lts__t_sectors_srcunit_tex_op_write.sum")
alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
l2info = {"l2_bytes_per_launch": None if l2 is None else l2 * 32, "l2_read_bytes": None if l2r is None else l2r * 32,
          "l2_write_bytes": None if l2w is None else l2w * 32, "algorithmic_bytes": alg,
          "l2_over_algorithmic": None if (l2 is None or not alg) else l2 * 32 / alg}
summary = {"report": rep, "metrics": d, "dram_bytes_per_launch": dram, "l2": l2info,
           "launch_list": {k: {"launches": len(v), "avg_ns": sum(v) / len(v), "share": sum(v) / tot} for k, v in agg.items()}}
json.dump(summary, open(out_prefix + ".json", "w"), indent=1)
with open(out_prefix + ".md", "w") as f:
    f.write(f"# ncu summary: {rep}\n\n| metric | value | unit |\n|---|---|---|\n")
    for k, v in d.items():
        f.write(f"| {k} | {v['value']} | {v['unit']} |\n")
    f.write(f"| dram bytes per launch (read+write) | {dram} | byte |\n")
    for k, v in l2info.items():
        f.write(f"| {k} | {v} | |\n")
    f.write("\n")
    f.write("## launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)\n\n")
    f.write("| kernel | launches | avg us | share of listed time |\n|---|---|---|---|\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"| {k} | {len(v)} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/tot:.3f} |\n")
print(json.dumps({k: v for k, v in summary.items() if k != "metrics"}, indent=1))
print({k: v["value"] + " " + v["unit"] for k, v in d.items()})
