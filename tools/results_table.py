"""Prints DESIGN.md §7's results table from the committed bench lines (profiles/r02/bench_*.json)."""
import json
import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]
ROWS = [("c5", "**C5 512³ 7-pt, p=8** (headline, wave)"), ("c1", "C1 64³ 7-pt, p=4"), ("c2", "C2 160³ 27-pt scrambled, p=8"),
        ("c3", "C3 R-MAT 21, p=4 (bitwise)"), ("c3fast", "C3 R-MAT 21, p=4 (fast)"),
        ("c4", "C4 192³ 27-pt Newton s=8"), ("c4poly", "C4 polynomial z = Σ c_k A^k x"),
        ("c4jac", "C4 s-step Jacobi basis (2 sweeps)"), ("c4gs2", "C4 s-step GS2 basis (γ=1, K=1)"),
        ("c4prod", "C4 degree-40 product-form polynomial"),
        ("c4ortho", "c4ortho: ICGS (2 sweeps, q=25) + TSQR (s=8), n=192³, fast")]


def main():
    print("| config | GF/s | step ms | roofline frac | per-power HBM frac | DRAM B/nnz: ncu / single pass / p passes | e2e GF/s | CPU baseline GF/s (kind, cores) | parity | clocks |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for key, name in ROWS:
        f = ROOT / "profiles" / "r02" / f"bench_{key}.json"
        if not f.exists():
            continue
        d = json.loads(f.read_text())
        r = d.get("roofline") or {}
        pp = (r.get("per_power") or {}).get("frac")
        e = d.get("e2e") or {}
        c = d.get("cpu_baseline") or {}
        par = d.get("parity") or d["config"].get("parity", "")
        if key == "c4ortho":
            par = "Q orthonormal, Q ⟂ basis, C vs bitwise ≤1e-12"
        else:
            par = "bitwise" if "bitwise" in par else ("≤1e-12" if "rel err" in par else par.split(" ")[0])
        cl = d.get("clocks") or {}
        print(f"| {name} | {d['value']:.1f} | {d['ms_per_step']:.3f} | {r.get('frac', 0):.3f} | "
              f"{pp:.2f} |" if pp is not None else f"| {name} | {d['value']:.1f} | {d['ms_per_step']:.3f} | "
              f"{r.get('frac', 0):.3f} | — |", end="")
        bn = [r.get("dram_bytes_per_nnz"), r.get("dram_bytes_per_nnz_single_pass"), r.get("dram_bytes_per_nnz_back_to_back")]
        bcell = " / ".join(f"{v:.1f}" if v else "—" for v in bn) if any(bn) else "—"
        print(f" {bcell} | {e.get('value', 0):.1f} | {c.get('value', 0):.2f} ({c.get('kind')}, {c.get('cores')}) | {par} | "
              f"{cl.get('sm_mhz')} MHz {','.join(cl.get('reasons') or []) or ''} |")


if __name__ == "__main__":
    main()
