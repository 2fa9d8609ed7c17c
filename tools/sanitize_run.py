"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): c1 doubly-iterative inverse power, a 4-system c4 complete-LU
inverse-power batch, the opt-in frontal LU on 2 systems, one SpMV, and a
'cmd'-ordered direct solve."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, factor, liouville, ordering, steady  # noqa: E402


def main():
    H, c = configs.kerr()
    L1 = liouville.build_liouvillian(H, c)
    r = steady.inverse_power(L1, tol=1e-12, inner="iterative", ordering_name="rcm",
                             solver="bicgstab", d=1e-5, p=10.0, seed=0)
    print("c1 power-bicgstab residual", r.residual)
    r = steady.solve_direct(L1, "cmd")
    print("c1 direct cmd residual", r.residual)
    L4 = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in (0, 100, 200, 300)])
    rs = steady.inverse_power_batch(L4, [2, 102, 202, 302], tol=1e-12, inner="direct",
                                    ordering_name="rcm")
    print("c4 batch residuals", [x.residual for x in rs])
    os.environ["RHOSOLVE_FRONTAL"] = "1"
    sh = liouville.shift(liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in (5, 9)]))
    fwd, inv = ordering.rcm_device(sh.matrix)
    f = factor.lu(ordering.permute(sh.matrix, fwd, inv))
    print("frontal fill", f.fill_factors)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
