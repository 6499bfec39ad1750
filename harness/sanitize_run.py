"""Small searches for compute-sanitizer (memcheck / racecheck / synccheck,
ONE tool per gpurun call -- B200_PROFILING.md): the golden cases `small` and
`sift_mini` through search_batch (K1 tensor-core + SIMT select, the
persistent warp-specialised scan kernel and the per-query scan kernel) for
every LUT dtype, checked against the reference goldens.  numpy + ctypes only
(no torch), so the sanitizer sees only this library's kernels.

  compute-sanitizer --tool memcheck python -m harness.sanitize_run
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2301_06672_b200 as pkg
    from paper_2301_06672_b200 import _lib
    z = {n: np.load(os.path.join(ROOT, "tests", "golden", f"{n}.npz")) for n in ("small", "sift_mini")}
    n_ok = 0
    for scan_mode in (0, 1):                       # persistent ws kernel, per-query kernel
        _lib.check(_lib.lib.ivfpq_set_scan_kernel(scan_mode))
        for sel_mode in (0, 1):                    # tensor-core K1 (auto), SIMT K1
            _lib.check(_lib.lib.ivfpq_set_select_kernel(sel_mode))
            for name, c in z.items():
                idx = pkg.IvfPqIndex.from_csr(c["coarse"], pkg.PQCodebook(centers=c["centers"], p=int(c["p"])),
                                              c["list_off"], c["ids"], c["codes"])
                P = 8 if name == "sift_mini" else 4
                for prec in ("f32", "f16", "e5m3", "e4m4"):
                    lists, _ = pkg.search_batch(idx, c["queries"], pkg.SearchParams(k=10, nprobe=P, precision=prec))
                    assert np.array_equal(lists.ids, c[f"ids_{prec}_k10_p{P}"]), (name, prec, scan_mode, sel_mode)
                    n_ok += 1
    _lib.check(_lib.lib.ivfpq_set_scan_kernel(0))
    _lib.check(_lib.lib.ivfpq_set_select_kernel(0))
    print(f"sanitize_run ok: {n_ok} searches bit-exact vs goldens")


if __name__ == "__main__":
    main()
