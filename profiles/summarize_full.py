"""Summarises an `ncu --set full` raw-page CSV (ncu -i X.ncu-rep --page raw
--csv): per kernel the duration, issue/pipe utilisation, occupancy, DRAM
traffic and throughput, shared-memory bank conflicts and the top stall
reasons."""
import csv
import sys


def f(d, k):
    try:
        return float(d.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    print(f"source: {path}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        dur = f(d, "gpu__time_duration.sum")
        rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
        print(f"\n{name}  grid {d.get('launch__grid_size')} x {d.get('launch__block_size')}  "
              f"cluster {d.get('launch__cluster_dim_x')}  regs {d.get('launch__registers_per_thread')}  "
              f"smem/CTA {d.get('launch__shared_mem_per_block')} KB")
        print(f"  duration {dur:.1f} us; DRAM read {rd:.1f} + write {wr:.1f} MB "
              f"({(rd + wr) / dur:.2f} TB/s = {f(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}% of peak)")
        print(f"  issue active {f(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}%  "
              f"warps active {f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%  "
              f"ALU {f(d, 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active'):.1f}%  "
              f"FMA(IMAD) {f(d, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%  "
              f"L2 hit {f(d, 'lts__t_sector_hit_rate.pct'):.1f}%")
        wf, ideal = f(d, "memory_l1_wavefronts_shared"), f(d, "memory_l1_wavefronts_shared_ideal")
        print(f"  smem wavefronts {wf:.0f} (ideal {ideal:.0f}, excess {100 * (wf / ideal - 1) if ideal else 0:.0f}%)  "
              f"instructions {f(d, 'smsp__inst_executed.sum'):.3g} warp-level")
        st = [(k, f(d, k)) for k in hdr if k.startswith("smsp__average_warps_issue_stalled")
              and k.endswith("per_issue_active.ratio")]
        st = sorted([x for x in st if x[1] == x[1]], key=lambda kv: -kv[1])[:6]
        print("  stalls per issue: " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for k, v in st))


if __name__ == "__main__":
    main(sys.argv[1])
