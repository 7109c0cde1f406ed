"""DRAM traffic per unit of work from `ncu --set full` raw-page CSVs
(`ncu -i X.ncu-rep --page raw --csv`), written to a JSON that bench.py reads
for `roofline.traffic`.

Units: key-switch kernels per ciphertext (the launch's ciphertext count is
recovered from its grid: ks_inner = count*(L+K)*CL CTAs, moddown =
count*2L*CL, input INTT = count*L*CL, P-limb INTT = count*2K*CL; the paired
kernels cover two ciphertexts, components or limbs per cluster), NTTs per
limb transform (grid = limbs*CL / transforms per cluster).

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
    res = {"source": "ncu --set full --clock-control none, launches inside one lola-mnist step "
                     "(tools/gpu_profile.sh); DRAM bytes = dram__bytes_read.sum + dram__bytes_write.sum",
           "params": {"L": L, "K": K, "cluster": CL}, "kernels": {}}
    acc = {}
    for path in sys.argv[5:]:
        for name, grid, rd, wr, dur in read(path):
            base = name.split("(")[0].replace("void ", "").replace("lb::", "").strip()
            pair = 2 if "_pair_" in base else 1
            if "ks_inner_mix" in base:
                # grid.x covers L + 2K virtual targets, grid.y ciphertext pairs
                unit, per, launches = "ciphertext", 2 * grid // ((L + 2 * K) * CL), 1
            elif "ks_inner" in base:
                unit, per, launches = "ciphertext", pair * grid // ((L + K) * CL), 1
            elif "moddown" in base:
                unit, per, launches = "ciphertext", pair * grid // (2 * L * CL), 1
            elif "ntt_" in base:
                # <LOGN, word, storage, mapped, transforms per cluster>; the key
                # switch's two inverse transforms (input: L limbs, P limbs of both
                # accumulators: 2K limbs) share one instance
                args = base[base.index("<") + 1:base.rindex(">")].split(",")
                nt = int(args[4]) if len(args) > 4 else 1
                unit, per, launches = "limb", nt * grid // CL, None
            else:
                unit, per, launches = "launch", 1, None
            a = acc.setdefault(base, {"unit": unit, "units": 0, "bytes": 0.0, "us": 0.0, "n": 0})
            a["units"] += per
            a["bytes"] += (rd + wr) * 1e6
            a["us"] += dur
            a["n"] += 1
    for base, a in acc.items():
        res["kernels"][base] = {"unit": a["unit"], "launches_captured": a["n"], "units_captured": a["units"],
                                "bytes_per_unit": a["bytes"] / a["units"], "mean_duration_us": a["us"] / a["n"]}
    # composite: DRAM bytes of one key switch per ciphertext
    per_ct = 0.0
    for base, v in res["kernels"].items():
        if "ks_inner" in base or "moddown" in base:
            per_ct += v["bytes_per_unit"]
        elif base.startswith("ntt_inverse_kernel<14, unsigned int, unsigned int"):
            per_ct += v["bytes_per_unit"] * (L + 2 * K)
    res["key_switch_bytes_per_ciphertext"] = per_ct
    json.dump(res, open(out_path, "w"), indent=1)
    for k, v in res["kernels"].items():
        print(f"{k:60s} {v['units_captured']:6d} {v['unit']:12s} {v['bytes_per_unit'] / 1e6:8.3f} MB/unit")
    print(f"key switch: {per_ct / 1e6:.3f} MB per ciphertext")


if __name__ == "__main__":
    main()
