"""Build profiles/r01_traffic.json from the `--set full` captures of tools/ncu_round.sh.

Per captured launch: DRAM read + write bytes (dram__bytes_read.sum / dram__bytes_write.sum) and the
duration; per op of bench.py (config 5, 2048^3, 1 GPU, W = 64): the DRAM bytes of one step = the
per-launch traffic x launches per step (HSZP_ND: 32 windows of band scan + z-sweep; HSZX_ND: one
fused launch).  bench.py reports it as roofline.traffic.

    python tools/traffic_json.py gpurun_out/full_k_band_scan.ncu-rep gpurun_out/full_k_zsweep_ring.ncu-rep \
        gpurun_out/full_k_fused_blocks.ncu-rep [--out profiles/r01_traffic.json]
"""

import argparse
import csv
import io
import json
import subprocess

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1.0}
VALUES = 64 * 2048 * 2048          # values per HSZP_ND window launch


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    get = {}
    for h, u, v in zip(head, units, vals):
        try:
            get[h] = float(v.replace(",", "")) * UNITS.get(u, 1.0)
        except ValueError:
            get[h] = v
    return get


def entry(path, launch, values):
    g = raw(path)
    rd, wr, t = g["dram__bytes_read.sum"], g["dram__bytes_write.sum"], g["gpu__time_duration.sum"]
    return {"kernel": g.get("Kernel Name", ""), "launch": launch, "values_per_launch": values,
            "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes_per_launch": rd + wr,
            "ncu_duration_s": t, "ncu_dram_gbs": (rd + wr) / t / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("band_scan")
    ap.add_argument("zsweep")
    ap.add_argument("fused")
    ap.add_argument("--out", default="profiles/r01_traffic.json")
    a = ap.parse_args()
    k = {
        "reconstruct:hszp-nd": entry(a.band_scan, "one 64-plane window (band scan, int8 L)", VALUES),
        "stencil:hszp-nd": entry(a.zsweep, "one 64-plane window of the 2048^3 HSZP_ND slab (int8 L)", VALUES),
        "fused:hszx-nd": entry(a.fused, "the whole 2048^3 HSZX_ND slab (one launch)", 2048 ** 3),
    }
    ops = {
        "hszp-nd": {"kernels": ["k_band_scan x32 (+ k_band_prefix, L2-resident)", "k_zsweep_ring x32"],
                    "traffic_bytes_per_step": int(32 * (k["reconstruct:hszp-nd"]["traffic_bytes_per_launch"]
                                                        + k["stencil:hszp-nd"]["traffic_bytes_per_launch"]))},
        "hszx-nd": {"kernels": ["k_fused_blocks x1"],
                    "traffic_bytes_per_step": int(k["fused:hszx-nd"]["traffic_bytes_per_launch"])},
    }
    with open(a.out, "w") as f:
        json.dump({"kernels": k, "ops": ops}, f, indent=1)
    print(json.dumps(ops, indent=1))


if __name__ == "__main__":
    main()
