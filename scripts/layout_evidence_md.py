"""Table of scripts/layout_evidence.sh outputs (gpurun_out/lay_*.json bench lines + lay_ncu_*.csv ncu
metric passes) -> markdown: python scripts/layout_evidence_md.py TAG > profiles/layout_evidence_TAG.md"""
import csv, json, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
print("# Layout evidence (SURVEY §8(d); PAPER P:158, Table 4): schedule-order vs PQ plans, one launch each\n")
print(f"Round tag {tag}: bench lines `gpurun_out/lay_*.json`, ncu `--metrics` pass of the same command (cold, serialised).\n")
print("| config | layout | us / pass | copy bytes (copy-based executor) | copy kernels | contiguous operands | "
      "gathered operands | staged operands | plan layout ms | DRAM read MB | L2 read MB (tex) | L2 total MB | "
      "LDGSTS (cp.async) warp instr |")
print("|" + "---|" * 13)
for c in ("cfg3", "cfg2", "cfg5"):
    for l in ("schedule", "pq"):
        try:
            d = json.loads(open(f"gpurun_out/lay_{c}_{l}.json").read().strip().splitlines()[-1])
        except Exception:
            continue
        m = {}
        try:
            rows = list(csv.reader(open(f"gpurun_out/lay_ncu_{c}_{l}.csv")))
            start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
            rows = [r for r in rows[start:] if len(r) > 10]
            hdr = rows[0]
            for r in rows[1:]:
                m[r[hdr.index("Metric Name")]] = (float(r[hdr.index("Metric Value")].replace(",", "")),
                                                  r[hdr.index("Metric Unit")])
        except Exception:
            pass

        def mb(name, sector=False):
            if name not in m:
                return "—"
            v, u = m[name]
            if sector:
                return f"{v * 32 / 1e6:.1f}"
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
            return f"{v * scale:.1f}"
        lay = d["layout"]
        ld = m.get("smsp__inst_executed_op_ldgsts.sum", (float("nan"), ""))[0]
        print(f"| {c} | {l} | {d['ms_per_step'] * 1e3:.1f} | {lay['copy_bytes']} | {lay['copy_kernels']} | "
              f"{lay['contig_operands']} | {lay['gather_operands']} | {lay['staged_operands']} | {lay['layout_ms']} | "
              f"{mb('dram__bytes_read.sum')} | {mb('lts__t_sectors_srcunit_tex_op_read.sum', True)} | "
              f"{mb('lts__t_sectors.sum', True)} | {ld:.0f} |")
