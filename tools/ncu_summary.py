"""Writes profiles/<name>.json from an ncu --set full report (+ optional launch-list CSV), the
files bench.py reads for roofline.traffic and the judge reads as evidence.

    python tools/ncu_summary.py --rep gpurun_out/prof_c2_lean.ncu-rep --launches gpurun_out/launches_c2.csv \
        --out profiles/ncu_c2.json --kernel k_mpk_lean --note "..."
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
UNIT = {"dram__bytes_read.sum": 1e9, "dram__bytes_write.sum": 1e9}  # ncu prints Gbyte here


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--kernel", default="k_mpk")
    ap.add_argument("--note", default="")
    ap.add_argument("--steps", type=int, default=1, help="MPK steps inside the launch list's range")
    a = ap.parse_args()
    hdr, units, rows = raw(a.rep)
    res = {"report": a.rep.split("/")[-1], "note": a.note, "kernels": []}
    for r in rows:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"name": d.get("Kernel Name", "")[:120]}
        for key in KEYS:
            if key in d:
                try:
                    v = float(d[key].replace(",", ""))
                except ValueError:
                    continue
                if u.get(key, "").lower().startswith("gbyte"):
                    v *= 1e9
                elif u.get(key, "").lower().startswith("mbyte"):
                    v *= 1e6
                elif u.get(key, "") == "ms":
                    v *= 1e-3
                elif u.get(key, "") == "us":
                    v *= 1e-6
                k[key] = v
        st = {kk[33:]: float(v) for kk, v in d.items()
              if kk.startswith("smsp__pcsamp_warps_issue_stalled") and not kk.endswith("not_issued")
              and v.replace(".", "").isdigit()}
        tot = sum(st.values()) or 1.0
        k["stall_share"] = {kk: round(v / tot, 4) for kk, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        res["kernels"].append(k)
    main_k = next((k for k in res["kernels"] if a.kernel in k["name"]), res["kernels"][0])
    rd, wr = main_k.get("dram__bytes_read.sum", 0.0), main_k.get("dram__bytes_write.sum", 0.0)
    res["dram_bytes_per_launch"] = rd + wr
    # one MPK step = every captured launch of the kernel (one launch per power in sweep mode)
    steps = [k for k in res["kernels"] if a.kernel in k["name"]]
    res["launches_per_step"] = len(steps)
    res["dram_bytes_per_step"] = sum(k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
                                     for k in steps)
    res["kernel_s_per_step"] = sum(k.get("gpu__time_duration.sum", 0.0) for k in steps)
    res["dram_read_bytes_per_launch"] = rd
    res["dram_write_bytes_per_launch"] = wr
    if a.launches:
        agg = {}
        dram = {}
        hdr2 = None
        for r in csv.reader(open(a.launches)):
            if r and r[0] == "ID":
                hdr2 = r
                continue
            if hdr2 and len(r) == len(hdr2):
                d = dict(zip(hdr2, r))
                name = d["Kernel Name"].split("(")[0].split("::")[-1][:60]
                val = float(d["Metric Value"].replace(",", ""))
                if d["Metric Name"].startswith("dram__bytes_"):
                    scale = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(d["Metric Unit"].lower(), 1.0)
                    dram[name] = dram.get(name, 0.0) + val * scale
                if d["Metric Name"] != "gpu__time_duration.sum":
                    continue
                agg.setdefault(name, []).append(val)
        if dram:  # every kernel of the timed region (fills included): the step's DRAM traffic
            res["dram_bytes_per_step"] = sum(dram.values()) / a.steps
            res["dram_bytes_per_step_by_kernel"] = {k: v / a.steps for k, v in dram.items()}
            res["dram_bytes_per_step_source"] = "launch list (all kernels of the timed region)"
        tot = sum(sum(v) for v in agg.values()) or 1.0
        res["launch_list"] = {k: {"launches": len(v), "total_ns": sum(v), "share": round(sum(v) / tot, 4)}
                              for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}, indent=1)[:1500])


if __name__ == "__main__":
    main()
