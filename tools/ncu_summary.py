"""Summarise an ncu --set full report as a markdown table (one row per profiled
kernel): duration, DRAM bytes and throughput, fp64 pipe, shared-memory
wavefronts, registers, occupancy, L2 hit rate and the top stall reasons.

    python tools/ncu_summary.py report.ncu-rep [> profiles/....md]
"""
import csv
import io
import subprocess
import sys


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def pick(h, r, *names):
    for nm in names:
        if nm in h:
            v = r[h.index(nm)]
            try:
                return float(v.replace(",", ""))
            except ValueError:
                return v
    return None


def main(path):
    h, u, rows = load(path)
    stall_cols = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued")]
    print("| kernel | duration ms | DRAM read GB | DRAM write GB | DRAM GB/s | fp64 pipe % | smem wavefronts % "
          "| regs | warps active % | L2 hit % | SM MHz | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        name = r[h.index("Kernel Name")]
        name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "").split("(")[0]
        t = pick(h, r, "gpu__time_duration.sum")
        tu = u[h.index("gpu__time_duration.sum")]
        t_ms = t / 1e6 if tu == "ns" else (t / 1e3 if tu == "us" else t)
        def gb(col):
            v = pick(h, r, col)
            un = u[h.index(col)]
            return v * {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "Tbyte": 1e3}.get(un, 1)
        rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
        fp64 = pick(h, r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
        smem = pick(h, r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")
        regs = pick(h, r, "launch__registers_per_thread")
        warps = pick(h, r, "sm__warps_active.avg.pct_of_peak_sustained_active")
        l2 = pick(h, r, "lts__t_sector_hit_rate.pct")
        clk = pick(h, r, "sm__cycles_elapsed.avg.per_second")
        clk_u = u[h.index("sm__cycles_elapsed.avg.per_second")] if "sm__cycles_elapsed.avg.per_second" in h else ""
        mhz = clk * {"Ghz": 1e3, "GHz": 1e3, "Mhz": 1, "MHz": 1, "hz": 1e-6}.get(clk_u, 1) if clk else None
        st = []
        for c in stall_cols:
            v = pick(h, r, c)
            if isinstance(v, float):
                st.append((v, c.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in st) or 1.0
        st.sort(reverse=True)
        top = ", ".join(f"{nm} {100 * v / tot:.0f}%" for v, nm in st[:3])
        fmt = lambda x, f="{:.1f}": f.format(x) if isinstance(x, float) else str(x)
        print(f"| {name} | {t_ms:.3f} | {rd:.2f} | {wr:.2f} | {(rd + wr) / t_ms * 1e3:.0f} | {fmt(fp64)} | {fmt(smem)} "
              f"| {fmt(regs, '{:.0f}')} | {fmt(warps)} | {fmt(l2)} | {fmt(mhz, '{:.0f}')} | {top} |")


if __name__ == "__main__":
    main(sys.argv[1])
