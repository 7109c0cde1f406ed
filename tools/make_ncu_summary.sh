# writes profiles/r02_ncu_full_keyswitch.txt from the CSV exports of tools/gpu_final_r2b.sh in gpurun_out/
cd "$(dirname "$0")/.."
OUT=profiles/r02_ncu_full_keyswitch.txt
{
echo "# r02 (final code): ncu --set full --clock-control none, launches inside one lola-mnist step at B=64 (tools/gpu_final_r2b.sh -> tools/gpu_profile.sh), 29-bit set, u32 residues; hot-path u32 NTTs from tools/ntt_launch.py (the bench's roofline_ntt launch)."
echo "# integer-pipe cross-check (tools/pipes.py): $(head -1 gpurun_out/r02_pipes.json)"
for f in full_1 full_2 full_3 full_ntt; do python profiles/summarize_full.py gpurun_out/$f.csv; done
python - <<'PY'
import csv
def num(x):
    try: return float(x.replace(",", ""))
    except Exception: return 0.0
for f in ("full_1", "full_2", "full_3", "full_ntt"):
    rows = list(csv.reader(open(f"gpurun_out/{f}.csv")))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        g = lambda k: d.get(k, "n/a")
        print(f"{d['Kernel Name'][:52]:52s} fmaheavy {g('sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active')}%  "
              f"lts {g('lts__t_sectors.avg.pct_of_peak_sustained_elapsed')}%  lsu {g('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active')}%")
PY
for f in source_1 source_2 source_3 source_ntt; do echo; python profiles/summarize_stalls.py gpurun_out/$f.csv | head -9; python profiles/summarize_fma.py gpurun_out/$f.csv | head -12; python tools/src_phases.py gpurun_out/$f.csv 1.5 | head -14; done
} > $OUT 2>&1
wc -l $OUT
