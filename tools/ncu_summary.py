"""Summarise ncu reports into a JSON + markdown table for profiles/ (run here, no GPU).
usage: python tools/ncu_summary.py out_prefix name=report.ncu-rep ..."""
import csv, io, json, subprocess, sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "gpc__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm_bytes",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_per_block",
    "launch__grid_size": "grid",
    "launch__cluster_size": "cluster",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_bank_conflicts_ld",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "smem_bank_conflicts_st",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum": "smem_st_wavefronts",
    "smsp__sass_inst_executed_op_shared_st.sum": "smem_st_instructions",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed": "l2_sector_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed": "l2_to_sm_pct_of_peak",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "compute_memory_throughput_pct",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    d = {"kernel": v[h.index("Kernel Name")]}
    for i, n in enumerate(h):
        if n in KEYS:
            val = v[i].replace(",", "")
            unit = u[i]
            try:
                x = float(val)
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "Tbyte": 1e12, "byte": 1, "Ghz": 1e9, "hz": 1,
                         "Mhz": 1e6, "us": 1, "ns": 1e-3, "ms": 1e3}.get(unit, 1)
                if KEYS[n] == "duration_us" and unit == "ns":
                    x = x / 1000.0
                elif KEYS[n] != "duration_us":
                    x = x * scale
                d[KEYS[n]] = x
            except ValueError:
                d[KEYS[n]] = val
    return d


def smem_excess(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[1]
    ix = {n: i for i, n in enumerate(h)}
    tot = ex = 0.0
    for row in r[2:]:
        if len(row) < len(h):
            continue
        try:
            tot += float(row[ix["L1 Wavefronts Shared"]] or 0)
            ex += float(row[ix["L1 Wavefronts Shared Excessive"]] or 0)
        except (ValueError, KeyError):
            pass
    return {"smem_wavefronts": tot, "smem_wavefronts_excessive": ex}


def main():
    prefix = sys.argv[1]
    res = {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        d = raw(rep)
        try:
            d.update(smem_excess(rep))
        except Exception as e:  # source page missing
            d["smem_note"] = str(e)
        res[name] = d
    with open(prefix + ".json", "w") as f:
        json.dump(res, f, indent=1)
    lines = ["| capture | kernel | us | SM GHz | tensor % | DRAM rd GB | DRAM wr GB | L2->SM GB | L2 hit % | L2 throughput % of peak | DRAM throughput % | regs | smem wavefronts excessive |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for n, d in res.items():
        lines.append(f"| {n} | `{d['kernel'][:60]}` | {d.get('duration_us', 0):.1f} | {d.get('sm_clock_hz', 0)/1e9:.3f} | "
                     f"{d.get('tensor_pipe_active_pct', 0):.1f} | {d.get('dram_read_bytes', 0)/1e9:.3f} | "
                     f"{d.get('dram_write_bytes', 0)/1e9:.3f} | {d.get('l2_to_sm_bytes', 0)/1e9:.2f} | "
                     f"{d.get('l2_hit_pct', 0):.1f} | {d.get('l2_throughput_pct', 'n/a')} | {d.get('dram_throughput_pct', 'n/a')} | "
                     f"{d.get('registers_per_thread', '')} | "
                     f"{d.get('smem_wavefronts_excessive', 'n/a')} of {d.get('smem_wavefronts', 'n/a')} |")
    with open(prefix + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
