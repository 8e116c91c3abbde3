"""Step-seam debug: plan-mode dots/coefficients of one step vs the oracle (cd2d16 trace)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from oracle import oracle as orc
    from paper_2108_10591_b200 import _lib
    from paper_2108_10591_b200.operators import DeviceMatrix
    from tests import golden_cases as gc

    spec, A, b, x0, g = gc.load_case("cd2d16", orc.spmv, trace=True)
    n = A.n_rows
    r0s = b.copy()
    coef = g["coef"]
    for mode in (0, 1):
     for i in range(0, 13):
        j = i + 1
        st = {k: g[f"it{i}_{k}"] for k in ("x", "r", "p", "u", "o", "t", "w", "y", "z", "s", "q", "g", "l")}
        st.update(r0s=r0s, b=b, As=np.zeros(n))
        r_prev = r0s if i == 0 else g[f"it{i - 1}_r"]
        f_prev = orc.plan_dot(r0s, r_prev, 1)
        order = ("x", "r", "p", "u", "o", "t", "w", "y", "z", "s", "q", "g", "l", "r0s", "b", "As")
        dm = DeviceMatrix.from_csr(A)
        dev = [torch.from_numpy(np.ascontiguousarray(st[k])).cuda() for k in order]
        ptrs = (C.c_void_p * 16)(*[t.data_ptr() for t in dev])
        sin = np.array([j, coef[i, 0], coef[i, 2], f_prev, float(g["r0_norm"]), 0.0])
        sout = np.zeros(14)
        _lib.check(_lib.load().pbs_step_dev(dm.handle, ptrs, sin.ctypes.data_as(C.c_void_p), mode, 1,
                                            sout.ctypes.data_as(C.c_void_p)), dm.ctx.handle)
        s, y, r, t = st["s"], st["y"], st["r"], st["t"]
        pairs = [(s, s), (y, y), (s, y), (s, r), (y, r), (r0s, r), (r0s, s), (r0s, t), (r, r)]
        ref_d = np.array([orc.plan_dot(a, bb, 1) for a, bb in pairs])
        q, al, be = orc.alpha_beta_safe(ref_d[5], f_prev, ref_d[6], ref_d[7], coef[i, 0], coef[i, 2], False)
        q2, z, e = orc.zeta_eta_safe(*ref_d[:5], False)
        print("mode", mode, "step", j, "dots==", np.array_equal(sout[4:13], ref_d), "coef-golden",
              (sout[:4] - coef[j]).tolist(), "oracle(same dots)-golden", (np.array([al, be, z, e]) - coef[j]).tolist(),
              "dot diffs", (sout[4:13] - ref_d).tolist() if not np.array_equal(sout[4:13], ref_d) else "")
        dm.free()


if __name__ == "__main__":
    main()
