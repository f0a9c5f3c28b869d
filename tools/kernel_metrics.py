"""profiles/r2_c4_kernel_metrics.json from the ncu metrics CSV of one c4 step
(tools/prof_r2.sh): per heavy kernel the duration and DRAM bytes of the step's
launches (the CholeskyQR2 setup's TN GEMMs are the first two gemm_tn_sym
launches and are skipped), plus the algorithmic bytes / flops the bench's
roofline uses."""
import csv
import io
import json
import sys
from collections import defaultdict

N, K = 256 ** 3, 400


def main():
    src, dst = sys.argv[1], sys.argv[2]
    text = open(src).read()
    rows = list(csv.reader(io.StringIO(text[text.find('"ID"'):])))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(dict)      # launch id -> metric -> value
    names = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        lid = int(r[ix["ID"]])
        names[lid] = r[ix["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        v = float(r[ix["Metric Value"]].replace(",", ""))
        u = r[ix["Metric Unit"]]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1.0)
        per[lid][r[ix["Metric Name"]]] = v * scale
    groups = defaultdict(list)
    for lid in sorted(per):
        groups[names[lid]].append(per[lid])
    out = {"config": "c4 256x256x256 K=400, one step (bench.py --profile-steps 1), ncu --metrics, --clock-control "
                     "none (serialised launches, cold caches: compare shares, not absolute times)", "kernels": {}}
    key = {"gemm_tn_sym_kernel": "projection_tn_sym", "stencil5_kernel": "stencil_delta",
           "reconstruct_dmma_kernel": "reconstruct_argmax", "oz_gemm_kernel": "rotation_int8_gemm",
           "oz_slice_rows_kernel": "rotation_digit_split"}
    for name, launches in groups.items():
        k = next((v for kk, v in key.items() if kk in name), None)
        if k is None:
            continue
        if k == "projection_tn_sym":
            launches = launches[2:]          # skip the setup's Gram matrices
        dur = sum(x.get("gpu__time_duration.sum", 0.0) for x in launches)
        rd = sum(x.get("dram__bytes_read.sum", 0.0) for x in launches)
        wr = sum(x.get("dram__bytes_write.sum", 0.0) for x in launches)
        ent = {"kernel": name, "launches": len(launches), "duration_ms": dur,
               "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
               "tensor_pipe_pct_elapsed": launches[0].get(
                   "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
               "l2_hit_pct": launches[0].get("lts__t_sector_hit_rate.pct")}
        if k.startswith("rotation"):
            # 16 launches (1M-row chunks) per c4 step; per-step traffic from the
            # mean launch when the capture holds fewer
            n_l = len(launches)
            ent["traffic_bytes_per_launch"] = (rd + wr) / n_l
            ent["traffic_bytes"] = (rd + wr) / n_l * 16
            ent["duration_ms_per_launch"] = dur / n_l
            ent["traffic_note"] = f"per step = 16 x the mean of the {n_l} captured launches"
        out["kernels"][k] = ent
    out["algorithmic"] = {"rotation_bytes": 16.0 * N * K, "stencil_bytes": 16.0 * N * K + 72.0 * N,
                          "projection_flops_sym": float(N) * K * (K + 1), "rotation_flops": 2.0 * N * K * K}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
