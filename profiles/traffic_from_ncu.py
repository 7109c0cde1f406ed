"""DRAM traffic per unit of work from `ncu --set full` raw-page CSVs
(`ncu -i X.ncu-rep --page raw --csv`), written to a JSON that bench.py reads
for `roofline.traffic`.

Units: key-switch kernels per ciphertext (the launch's ciphertext count is
recovered from its grid: ks_inner = count*(L+K)*CL CTAs, moddown =
count*2L*CL, input INTT = count*L*CL, P-limb INTT = count*2K*CL), NTTs per
limb transform (grid = limbs*CL).

usage: python traffic_from_ncu.py OUT.json L K CL full_1.csv full_2.csv ...
"""
import csv
import json
import sys


def read(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))

        def mb(k):
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[u[k]]
            return float(d[k].replace(",", "")) * scale

        out.append((d["Kernel Name"], int(d["launch__grid_size"]), mb("dram__bytes_read.sum"),
                    mb("dram__bytes_write.sum"), float(d["gpu__time_duration.sum"].replace(",", ""))))
    return out


def main():
    out_path, L, K, CL = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    res = {"source": "ncu --set full --clock-control none, one launch per kernel inside one lola-mnist step "
                     "(tools/gpu_profile.sh); DRAM bytes = dram__bytes_read.sum + dram__bytes_write.sum",
           "params": {"L": L, "K": K, "cluster": CL}, "kernels": {}}
    for path in sys.argv[5:]:
        for name, grid, rd, wr, dur in read(path):
            base = name.split("(")[0]
            if "ks_inner" in base:
                unit, per = "ciphertext", grid // ((L + K) * CL)
            elif "moddown" in base:
                unit, per = "ciphertext", grid // (2 * L * CL)
            elif "ntt_inverse_kernel" in base and "unsigned int, unsigned int" in base:
                unit, per = "ciphertext (2K P limbs)", grid // (2 * K * CL)
            elif "ntt_inverse_kernel" in base and "unsigned int, unsigned long" in base:
                unit, per = "ciphertext (L input limbs)", grid // (L * CL)
            elif "ntt_" in base:
                unit, per = "limb", grid // CL
            else:
                unit, per = "launch", 1
            res["kernels"][base] = {"unit": unit, "units_in_launch": per, "dram_read_mb": rd, "dram_write_mb": wr,
                                    "bytes_per_unit": (rd + wr) * 1e6 / per, "duration_us": dur}
    json.dump(res, open(out_path, "w"), indent=1)
    for k, v in res["kernels"].items():
        print(f"{k:60s} {v['units_in_launch']:5d} {v['unit']:28s} {v['bytes_per_unit'] / 1e6:8.3f} MB/unit")


if __name__ == "__main__":
    main()
