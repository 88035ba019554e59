"""Prints a one-line summary of bench.py JSON outputs (for quick reading of gpurun results)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    if "roofline" not in d:
        print(f, json.dumps(d)[:300])
        continue
    c, r = d["config"], d["roofline"]
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    print(f"{f}: {d['value']:.1f} GF/s step={d['ms_per_step']:.3f}ms kernel={r['kernel_ms']:.3f}ms "
          f"frac={r['frac']:.3f} achieved={r['achieved']:.0f}GB/s traffic={r.get('traffic')} "
          f"base={c.get('baseline_gflops', 0):.1f}GF/s ({c.get('baseline_back_to_back_ms', 0):.3f}ms) "
          f"{c.get('parity')} e2e={e2e.get('value', 0):.1f} cpu={cpu.get('value')} "
          f"launches={d.get('gpu_launches')} clk={d.get('clocks', {}).get('sm_mhz')} "
          f"exec={c.get('executor')}")
