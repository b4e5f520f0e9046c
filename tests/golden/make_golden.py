"""Generate tests/golden/golden.npz from the REFERENCE ITSELF.

Runs in the build container only (needs /root/reference, via the shim
oracle/_ref/librdmm_ref.so compiled by oracle/Makefile from the unmodified
reference headers).  The fixtures pin both the plain-C oracle restatement
(tests/test_oracle.py) and the CUDA path (tests/test_*_gpu.py).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402

VARIANTS = list(oracle.VARIANTS)
# (m, k, n, p, d, w, spgemm, flops, out_nnz): cfg3 SpMM at 1/4 GPUs, cfg5 at 2,
# a fp64 case, cfg4 SpGEMM at 8 (survey-measured flops / output nnz)
MODEL_CASES = [(4194304, 4194304, 128, 1, 64827941 / 4194304**2, 4, 0, 0, 0),
               (4194304, 4194304, 128, 4, 64827941 / 4194304**2, 4, 0, 0, 0),
               (4194304, 4194304, 256, 2, 16 / 4194304, 4, 0, 0, 0),
               (65536, 65536, 128, 9, 490332 / 65536**2, 8, 0, 0, 0),
               (1048576, 1048576, 1048576, 8, 8124707 / 1048576**2, 4, 1, 4696097190,
                1390953199)]
MODEL_COST = [900e9, 900e9, 6446.3e9, 74.4e12]


def csr(out, name, c):
    out[name + "_rp"] = c.row_ptr
    out[name + "_ci"] = c.col_idx
    out[name + "_v"] = c.values


def main():
    oracle.build()
    R = oracle.ref()
    g = {}
    # gen.hpp KATs (test_gen_io.cpp:44 pins splitmix64(0))
    g["kat_splitmix0"] = np.array([R.splitmix64(0)], dtype=np.uint64)
    R.lib.ref_rng_at.restype = oracle.C.c_uint64
    R.lib.ref_rng_at.argtypes = [oracle.C.c_uint64, oracle.C.c_uint64]
    g["kat_rng_at_1"] = np.array([R.lib.ref_rng_at(1, i) for i in range(8)], dtype=np.uint64)
    csr(g, "rmat10", R.rmat(10, 8, seed=1))
    csr(g, "rmat10m", R.rmat(10, 8, seed=1, multiplicity=True))
    csr(g, "unif64", R.uniform_tiles(64, 64, 4, 0.25, 3))
    csr(g, "rcsr", R.random_csr(24, 20, 0.25, 6))
    g["rdense"] = R.random_dense(20, 28, 7)
    csr(g, "perm8", R.permute_symmetric(R.rmat(8, 8, seed=1), 5))

    # spmm_local (tile.hpp:170-188), integer-valued and real-valued twins
    a = R.rmat(10, 8, seed=1)
    b = R.random_dense(a.cols, 16, 2)
    c = np.zeros((a.rows, 16), np.float32)
    g["spmm_flops"] = np.array([R.spmm_local(a, b, c)], dtype=np.uint64)
    g["spmm_b"] = b
    g["spmm_c"] = c
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        ar = oracle.Csr(a.rows, a.cols, a.row_ptr, a.col_idx, oracle.real_twin(a.nnz, 3, dt))
        br = oracle.real_twin(a.cols * 16, 4, dt).reshape(a.cols, 16)
        cr = oracle.real_twin(a.rows * 16, 5, dt).reshape(a.rows, 16)
        R.spmm_local(ar, br, cr)
        g["spmm_real_c_" + tag] = cr

    # spgemm_local (tile.hpp:211-255) on R-MAT s9 squared
    a9 = R.rmat(9, 8, seed=1)
    c9, fl = R.spgemm_local(a9, a9)
    csr(g, "spgemm9", c9)
    g["spgemm9_flops"] = np.array([fl], dtype=np.uint64)
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        ar = oracle.Csr(a9.rows, a9.cols, a9.row_ptr, a9.col_idx,
                        oracle.real_twin(a9.nnz, 3, dt))
        cr, _ = R.spgemm_local(ar, ar)
        g["spgemm9_real_v_" + tag] = cr.values
    # cancelled zeros stay (test_kernels.cpp:149-157)
    # csr_add (tile.hpp:257-288)
    x = R.random_csr(9, 7, 0.3, 23, dtype=np.float64)
    y = R.random_csr(9, 7, 0.3, 29, dtype=np.float64)
    csr(g, "csradd_x", x)
    csr(g, "csradd_y", y)
    csr(g, "csradd", R.csr_add(x, y))

    # run_multiply (algos.hpp:673-752), test_algos.cpp:17-18 shape, 2x2 grid
    kM, kK, kN, tm, tk, tn = 12, 9, 10, 4, 3, 4
    ga = R.random_csr(kM, kK, 0.35, 5, dtype=np.float64)
    gb = R.random_dense(kK, kN, 6, dtype=np.float64)
    gc0 = R.random_dense(kM, kN, 7, dtype=np.float64)
    outs = []
    for v in VARIANTS:
        c = gc0.copy()
        rep = R.run_multiply_spmm(ga, gb, c, variant=v, grid=(2, 2), tiles=(tm, tk, tn))
        outs.append((c, rep.checksum, rep.total_multiplies))
    for c, cs, mu in outs:
        assert np.array_equal(c, outs[0][0]) and cs == outs[0][1] and mu == 3 * 3 * 3
    g["algo_spmm_c"] = outs[0][0]
    g["algo_spmm_checksum"] = np.array([outs[0][1]])
    ga2 = R.random_csr(kM, kK, 0.35, 15, dtype=np.float64)
    gb2 = R.random_csr(kK, kN, 0.35, 16, dtype=np.float64)
    gc2 = R.random_csr(kM, kN, 0.15, 17, dtype=np.float64)
    outs = []
    for v in VARIANTS:
        c, rep = R.run_multiply_spgemm(ga2, gb2, gc2, variant=v, grid=(2, 2), tiles=(tm, tk, tn))
        outs.append((c, rep.checksum))
    for c, cs in outs:
        assert np.array_equal(c.col_idx, outs[0][0].col_idx)
        assert np.array_equal(c.values, outs[0][0].values) and cs == outs[0][1]
    csr(g, "algo_spgemm", outs[0][0])
    g["algo_spgemm_checksum"] = np.array([outs[0][1]])
    # analytics.hpp:66-150: predicted stage imbalance of A*A and the flop-table reduction
    a10 = R.rmat(10, 8, seed=1)
    for grid, stages in ((2, 0), (2, 4), (3, 6)):
        r = R.stage_imbalance(a10, grid, stages)
        key = f"stage_g{grid}s{stages}"
        g[key + "_flops"] = r["stage_flops"]
        g[key + "_imb"] = np.array([r["per_stage_flop_imbalance"],
                                    r["end_to_end_flop_imbalance"], r["nnz_imbalance"]])
    tab = np.random.default_rng(5).integers(0, 1000, size=(5, 7)).astype(np.uint64)
    tab[2] = 0
    g["imb_table"] = tab.astype(np.int64)
    r = R.imbalance_from_flops(tab)
    g["imb_table_out"] = np.array([r["per_stage_flop_imbalance"], r["end_to_end_flop_imbalance"]])
    # model.hpp:139-160 roofline at the BASELINE configs' shapes with B200 costs
    rows = []
    for m, k, n, p, d, w, sg, fl, on in MODEL_CASES:
        rows.append(R.roofline([m, k, n, p, d, w], MODEL_COST, sg, fl, on))
    g["model_out"] = np.array(rows)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **g)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
