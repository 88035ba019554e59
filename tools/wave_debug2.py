import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2309_02228_b200 as mpkg
from oracle.oracle import Oracle
from test_gpu_parity import corpus, DEFAULT_KNOBS
O = Oracle()
ctx = mpkg.Context(0)
for k, v in {**DEFAULT_KNOBS, "order": 0, "schedule": 3}.items():
    ctx.set_param(k, v)
for name in ("rmat_12", "stencil27_scrambled_20", "rmat_12"):
    A = corpus()[name]
    lv, pm, ip, lp = O.build_levels(A.row_ptr, A.col_idx)
    prp, pci, pv = O.permute(A.row_ptr, A.col_idx, A.values, pm)
    P = mpkg.HostCsr.from_arrays(prp, pci, pv)
    for src in ("host", "gpu"):
        Ap = ctx.csr(P)
        if src == "host":
            ls = ctx.levels_from_host(lv, pm, ip, lp)
        else:
            dA = ctx.csr(A); ls = ctx.build_levels(dA)
        x = mpkg.random_vector(P.n_rows, 9)
        plan = ctx.group_levels(ls, Ap, 1 << 20, 6)
        ref = O.baseline_mpk(prp, pci, pv, x, 6)
        got = ctx.mpk(plan, Ap, x, 6).as_matrix()
        bad = [int(np.count_nonzero(got[k].view(np.uint64) != ref[k].view(np.uint64))) for k in range(7)]
        print(name, src, plan.exec_info(), bad, "levels", ls.n_levels(), len(lp) - 1, flush=True)
