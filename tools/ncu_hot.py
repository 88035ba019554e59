"""Summarises an ncu report: key metrics, stall reasons, and the hottest SASS instructions.

    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [kernel_index]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, d = rows[0], dict(zip(rows[0], rows[2 + kidx]))
print("kernel:", d.get("Kernel Name", "")[:100])
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
          "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
          "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
          "launch__grid_size", "launch__block_size"]:
    print(f"  {k:55s} {d.get(k)}")
st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled")
      and not k.endswith("not_issued") and v.replace(".", "").isdigit()]
tot = sum(v for _, v in st) or 1
print("stalls:", ", ".join(f"{k[33:]}={100 * v / tot:.1f}%" for k, v in sorted(st, key=lambda x: -x[1])[:7]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
blocks, cur = [], None
for r in srows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
    elif cur is not None:
        cur.append(r)
if blocks:
    b = blocks[min(kidx, len(blocks) - 1)]
    h = b[0]
    ia, sa = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in b[1:] if len(r) > sa and r[sa].isdigit()]
    ts = sum(int(r[sa]) for r in data) or 1
    ti = sum(int(r[ia]) for r in data if r[ia].isdigit()) or 1
    print("hot SASS (stall share / inst share):")
    for r in sorted(data, key=lambda r: -int(r[sa]))[:25]:
        print(f"  {r[0][-5:]} {100 * int(r[sa]) / ts:5.1f}% {100 * int(r[ia]) / ti:5.1f}%  {r[1].strip()[:70]}")
