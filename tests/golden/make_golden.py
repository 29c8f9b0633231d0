"""Generate the golden parity fixtures by running the REAL reference.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py

Every case stores the inputs it was fed (or the seed recipe plus a sha256 of
the bytes when the input is large and regenerable with plain numpy) and the
reference outputs. The fixtures travel with the repo; nothing at test time
reads /root/reference.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np
import scipy.sparse as sp

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def uniform_x(m, n, seed):
    """cfg1-style input: fp32-representable uniform values."""
    return np.random.default_rng(seed).random((m, n, n), dtype=np.float32)


def main():
    sys.path.insert(0, REF)
    import rescalkit as rk
    from rescalkit.dist_rescal import perturbation_field

    out = {}

    # 1. config 1: dense m=8, n=256, k=4, 200 tracked iterations, fp64 oracle on
    #    fp32-representable X with random_init(256, 4, 8, 0) as the start.
    x32 = uniform_x(8, 256, 0)
    x = rk.RelTensor(x32.astype(np.float64))
    f0 = rk.random_init(256, 4, 8, 0)
    f, tr = rk.rescal_solve(x, 4, rk.SolverConfig(max_iters=200), initial=f0)
    out["cfg1_uniform"] = dict(x_recipe=np.array([8, 256, 0]), x_sha=_sha(x32), A0=f0.A, R0=f0.R,
                               A=f.A, R=f.R, trace=tr)
    fu, tru = rk.rescal_solve(x, 4, rk.SolverConfig(max_iters=200, track_error=False), initial=f0)
    out["cfg1_untracked"] = dict(A=fu.A, R=fu.R, trace_len=np.array(len(tru)))

    # 2. planted, lightly noised (synth.generate), small enough to store X
    xp, ap, rp = rk.generate(rk.SynthSpec(n=64, m=4, k_true=4, noise=0.01, seed=1))
    f0p = rk.random_init(64, 4, 4, 3)
    fp, trp = rk.rescal_solve(xp, 4, rk.SolverConfig(max_iters=300), initial=f0p)
    out["planted64"] = dict(X=xp.slices, A0=f0p.A, R0=f0p.R, A=fp.A, R=fp.R, trace=trp)

    # 3. exact recovery with a tolerance stop (test_rescal.py:119-122 shape)
    xe, _, _ = rk.generate(rk.SynthSpec(n=16, m=4, k_true=3, noise=0.0, seed=1, pedestal=0.15))
    fe, tre = rk.rescal_solve(xe, 3, rk.SolverConfig(max_iters=2000, tolerance=1e-4, seed=11))
    fe0 = rk.random_init(16, 3, 4, 11)
    out["exact16_tol"] = dict(X=xe.slices, A0=fe0.A, R0=fe0.R, A=fe.A, R=fe.R, trace=tre)

    # 4. all-ones rank one (test_rescal.py:110-117)
    xo = rk.RelTensor(np.ones((1, 2, 2)))
    fo, tro = rk.rescal_solve(xo, 1, rk.SolverConfig(max_iters=2000, tolerance=1e-8, seed=3))
    no = rk.finalize_normalize(fo)
    out["all_ones"] = dict(X=xo.slices, A=fo.A, R=fo.R, trace=tro, An=no.A, Rn=no.R)

    # 5. split API single steps and rel_error on a small random tensor
    rng = np.random.default_rng(27)
    xs = rng.random((3, 7, 7))
    f0s = rk.random_init(7, 2, 3, 28)
    fr = rk.update_r(rk.RelTensor(xs), f0s)
    fa = rk.update_a(rk.RelTensor(xs), f0s)
    fsplit = rk.update_a(rk.RelTensor(xs), fr)
    out["split7"] = dict(X=xs, A0=f0s.A, R0=f0s.R, R_upd=fr.R, A_upd=fa.A, A_split=fsplit.A,
                         R_split=fsplit.R, rel_err=np.array(rk.rel_error(rk.RelTensor(xs), f0s)))

    # 6. fp32 end-to-end (test_rescal.py:150-154)
    x32s = np.random.default_rng(12).random((2, 8, 8)).astype(np.float32)
    f32, tr32 = rk.rescal_solve(rk.RelTensor(x32s), 2, rk.SolverConfig(max_iters=20, seed=1))
    out["fp32_small"] = dict(X=x32s, A=f32.A, R=f32.R, trace=tr32)

    # 7. regress_r / rel_error with frozen A (test_rescal.py:249-254 shape)
    xr, ar, rr = rk.generate(rk.SynthSpec(n=16, m=3, k_true=3, noise=0.0, seed=21))
    rfit = rk.regress_r(xr, ar)
    out["regress16"] = dict(X=xr.slices, A=ar, R_true=rr, R_fit=rfit,
                            err=np.array(rk.rel_error(xr, rk.RescalFactors(ar, rfit))))

    # 8. finalize_normalize
    fn0 = rk.random_init(9, 3, 2, 17)
    fn = rk.finalize_normalize(fn0)
    out["normalize"] = dict(A0=fn0.A, R0=fn0.R, A=fn.A, R=fn.R)

    # 9. perturbation field / perturb (dense and sparse)
    pc = rk.PerturbConfig(delta=0.02, base_seed=5)
    fld = perturbation_field(9, 2, pc, (3, 4))
    xd = np.random.default_rng(11).random((2, 9, 9))
    pdense = rk.perturb(rk.RelTensor(xd), pc, (3, 4))
    xsp = rk.sparsify(rk.RelTensor(xd), 0.3)
    psp = rk.perturb(xsp, pc, (3, 4))
    out["perturb9"] = dict(field=fld, X=xd, Xp=pdense.slices,
                           sp_indptr=np.stack([s.indptr for s in xsp.slices]),
                           sp_indices=np.concatenate([s.indices for s in xsp.slices]),
                           sp_data=np.concatenate([s.data for s in xsp.slices]),
                           sp_nnz=np.array([s.nnz for s in xsp.slices]),
                           psp_data=np.concatenate([s.data for s in psp.slices]),
                           psp_indices=np.concatenate([s.indices for s in psp.slices]))

    # 10. CSR canonicalisation: duplicates, explicit zeros, unsorted columns
    r_ = np.array([0, 0, 1, 2, 2, 2, 3, 3, 0])
    c_ = np.array([2, 1, 0, 3, 3, 1, 0, 0, 2])
    v_ = np.array([1.0, 2.0, 0.0, 0.5, 0.25, 3.0, 1.0, -1.0, 4.0])
    coo = sp.coo_matrix((v_, (r_, c_)), shape=(4, 4))
    canon = rk.SparseRelTensor([coo]).slices[0]
    out["csr_canon"] = dict(rows=r_, cols=c_, vals=v_, indptr=canon.indptr, indices=canon.indices,
                            data=canon.data)

    # 11. sparse solve equals dense solve (test_dist_rescal.py:190-198 shape)
    xsd = rk.sparsify(rk.RelTensor(np.random.default_rng(14).random((2, 12, 12))), 0.15)
    fs_, ts_ = rk.rescal_solve(xsd, 2, rk.SolverConfig(max_iters=40, seed=3))
    fs0 = rk.random_init(12, 2, 2, 3)
    out["sparse12"] = dict(X=xsd.to_dense().slices, A0=fs0.A, R0=fs0.R, A=fs_.A, R=fs_.R, trace=ts_)

    # 12. grid solve p=4 with padding (test_dist_rescal.py:55-63 shape)
    xg = rk.RelTensor(np.random.default_rng(3).random((2, 7, 7)))
    fg, tg, _ = rk.solve_on_grid(xg, 2, rk.SolverConfig(max_iters=40, seed=4), 4)
    out["grid7_p4"] = dict(X=xg.slices, A=fg.A, R=fg.R, trace=tg)

    # 13. RESCALk on a planted tensor (test_model_select.py:270-282 shape)
    xk, _, _ = rk.generate(rk.SynthSpec(n=16, m=3, k_true=3, noise=0.01, seed=5))
    rep = rk.rescalk(xk, 2, 4, r=4, cfg=rk.SolverConfig(max_iters=120, seed=6),
                     pcfg=rk.PerturbConfig(delta=0.02, base_seed=6))
    out["rescalk16"] = dict(
        X=xk.slices, k_opt=np.array(rep.k_opt), low_conf=np.array(rep.low_confidence),
        ks=np.array([e.k for e in rep.entries]),
        s_min=np.array([e.s_min for e in rep.entries]),
        s_avg=np.array([e.s_avg for e in rep.entries]),
        rel_error=np.array([e.rel_error for e in rep.entries]),
        **{f"medians_k{e.k}": e.medians for e in rep.entries},
        **{f"core_k{e.k}": e.core for e in rep.entries},
    )

    # 14. the planted inputs of the reference's own tests (synth.generate), so
    #     the device test bodies run on identical data
    planted = {
        "p16_4_3_s1_ped": dict(n=16, m=4, k_true=3, seed=1, noise=0.0, pedestal=0.15),
        "p16_2_2_s3_ped": dict(n=16, m=2, k_true=2, seed=3, noise=0.0, pedestal=0.15),
        "p16_3_3_s7_ped": dict(n=16, m=3, k_true=3, seed=7, noise=0.0, pedestal=0.15),
        "p8_2_2_s9": dict(n=8, m=2, k_true=2, seed=9, noise=0.01),
        "p12_2_2_s10": dict(n=12, m=2, k_true=2, seed=10, noise=0.01),
    }
    pl = {}
    for key, spec in planted.items():
        xt, at, rt = rk.generate(rk.SynthSpec(**spec))
        pl[f"{key}_X"] = xt.slices
    rep7 = rk.rescalk(rk.RelTensor(pl["p16_3_3_s7_ped_X"]), 3, 3, r=2, cfg=rk.SolverConfig(max_iters=600, seed=8),
                      pcfg=rk.PerturbConfig(delta=0.01, base_seed=8))
    pl["p16_3_3_s7_ped_rescalk_s_min"] = np.array(rep7.entries[0].s_min)
    pl["p16_3_3_s7_ped_rescalk_rel_error"] = np.array(rep7.entries[0].rel_error)
    out["planted_inputs"] = pl

    # 15. NNDSVD start (rescal.py:327-372): dense full-SVD branch and the sparse
    #     ARPACK svds branch, on the planted tensor of case 2 (well separated
    #     leading singular values), plus a short nndsvd-initialised solve
    fn = rk.nndsvd_init(xp, 4)
    fs, trs = rk.rescal_solve(xp, 4, rk.SolverConfig(max_iters=50, init="nndsvd"))
    xsp2 = rk.sparsify(xp, 0.9)  # no all-zero rows: u has no structural zeros
    fsp = rk.nndsvd_init(xsp2, 3)
    out["nndsvd64"] = dict(X=xp.slices, A=fn.A, R=fn.R, A50=fs.A, R50=fs.R, trace50=trs,
                           sp_indptr=np.stack([q.indptr for q in xsp2.slices]),
                           sp_indices=np.concatenate([q.indices for q in xsp2.slices]),
                           sp_data=np.concatenate([q.data for q in xsp2.slices]),
                           sp_nnz=np.array([q.nnz for q in xsp2.slices]), spA=fsp.A, spR=fsp.R)

    # 16. %rescalk-coo ingest (tensor.py:249-300): a file written by the
    #     reference's save_tensor, a hand-written unsorted one with duplicates,
    #     explicit zeros and blank lines, and malformed files with the
    #     reference's error messages
    import tempfile
    from rescalkit.errors import DataError as RefDataError
    texts = {}
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "x.coo")
        rk.save_tensor(xsp2, path)
        texts["saved"] = open(path, encoding="utf-8").read()
    texts["messy"] = ("%rescalk-coo 5 2 9\n"
                      "1 4 0 2.5\n0 3 3 1e-3\n\n0 0 4 0.0\n1 4 0 0.25\n  0 3 1   7 \n"
                      "1 2 2 +3\n0 3 3 0.125\n1 0 0 inf\n0 1 1 1.5e+2\n")
    bad = {
        "bad_header": "%rescalk-co 3 1 1\n0 0 0 1.0\n",
        "bad_fields": "%rescalk-coo 3 1 2\n0 0 0 1.0\n0 1 1\n",
        "bad_relation": "%rescalk-coo 3 1 1\n1 0 0 1.0\n",
        "bad_index": "%rescalk-coo 3 1 1\n0 0 3 1.0\n",
        "bad_negative": "%rescalk-coo 3 1 1\n0 0 1 -2.0\n",
        "bad_count": "%rescalk-coo 3 1 3\n0 0 1 2.0\n0 1 1 2.0\n",
        "bad_float": "%rescalk-coo 3 1 1\n0 0 1 abc\n",
    }
    coo = {}
    with tempfile.TemporaryDirectory() as td:
        for name, txt in list(texts.items()) + list(bad.items()):
            path = os.path.join(td, name + ".coo")
            with open(path, "w", encoding="utf-8") as fh:
                fh.write(txt)
            coo[f"{name}_text"] = np.array(txt)
            try:
                tt = rk.load_tensor(path)
            except RefDataError as ex:
                coo[f"{name}_error"] = np.array(str(ex))
                continue
            coo[f"{name}_n"] = np.array(tt.n)
            for t, sl in enumerate(tt.slices):
                coo[f"{name}_indptr{t}"] = sl.indptr
                coo[f"{name}_indices{t}"] = sl.indices
                coo[f"{name}_data{t}"] = sl.data
    out["coo_ingest"] = coo

    import numpy, scipy
    meta = dict(numpy=numpy.__version__, scipy=scipy.__version__, reference=REF)
    for name, d in out.items():
        d = dict(d)
        d["meta"] = np.array(repr(meta))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print("wrote", name)


def extra_cases(names):
    """Round-2 fixtures, written one by one (``make_golden.py <name> ...``)
    so the earlier fixtures are not rewritten."""
    sys.path.insert(0, REF)
    import rescalkit as rk
    import tempfile

    meta = np.array(repr(dict(numpy=np.__version__, scipy=sp.__version__ if hasattr(sp, "__version__") else "",
                              reference=REF)))
    if "rescalk_cfg5" in names:
        # cfg5's sweep shape (k = 2..16, r = 10, delta = 0.02, 200 iterations,
        # SolverConfig defaults otherwise) at a host-affordable n: a planted
        # k_true = 6 tensor, m = 8 (model_select.py:422-503)
        x, _, _ = rk.generate(rk.SynthSpec(n=256, m=8, k_true=6, noise=0.01, seed=21))
        rep = rk.rescalk(x, 2, 16, r=10, cfg=rk.SolverConfig(max_iters=200, seed=0),
                         pcfg=rk.PerturbConfig(delta=0.02, base_seed=0))
        d = dict(X=x.slices, k_opt=np.array(rep.k_opt), low_conf=np.array(rep.low_confidence),
                 ks=np.array([e.k for e in rep.entries]),
                 s_min=np.array([e.s_min for e in rep.entries]),
                 s_avg=np.array([e.s_avg for e in rep.entries]),
                 rel_error=np.array([e.rel_error for e in rep.entries]), meta=meta)
        np.savez_compressed(os.path.join(HERE, "rescalk_cfg5.npz"), **d)
        print("wrote rescalk_cfg5", rep.k_opt, [round(e.s_min, 4) for e in rep.entries])
    if "rescalk_sparse" in names:
        # RESCALk on a SparseRelTensor: the reference resamples the stored
        # values only (dist_rescal.py:205-214, model_select.py:450)
        xp, _, _ = rk.generate(rk.SynthSpec(n=64, m=3, k_true=3, noise=0.01, seed=23))
        xs = rk.sparsify(xp, 0.4)
        rep = rk.rescalk(xs, 2, 4, r=4, cfg=rk.SolverConfig(max_iters=150, seed=2),
                         pcfg=rk.PerturbConfig(delta=0.02, base_seed=5))
        d = dict(X=xs.to_dense().slices, k_opt=np.array(rep.k_opt), ks=np.array([e.k for e in rep.entries]),
                 s_min=np.array([e.s_min for e in rep.entries]), s_avg=np.array([e.s_avg for e in rep.entries]),
                 rel_error=np.array([e.rel_error for e in rep.entries]),
                 **{f"medians_k{e.k}": e.medians for e in rep.entries}, meta=meta)
        np.savez_compressed(os.path.join(HERE, "rescalk_sparse.npz"), **d)
        print("wrote rescalk_sparse", rep.k_opt, [round(e.s_min, 4) for e in rep.entries])
    if "io_bytes" in names:
        # the reference writer's exact bytes for a dense f32 / f64 tensor, a
        # factor matrix and a COO file (tensor.py:188-327)
        rng = np.random.default_rng(31)
        d = {}
        with tempfile.TemporaryDirectory() as td:
            for tag, dt in (("f32", np.float32), ("f64", np.float64)):
                xt = rk.RelTensor(rng.random((3, 9, 9)).astype(dt))
                path = os.path.join(td, f"{tag}.rsk")
                rk.save_tensor(xt, path)
                d[f"dense_{tag}_X"] = xt.slices
                d[f"dense_{tag}_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
            a = rng.random((11, 4))
            path = os.path.join(td, "a.rskm")
            rk.save_matrix(a, path)
            d["matrix_A"] = a
            d["matrix_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
            xs = rk.sparsify(rk.RelTensor(rng.random((2, 10, 10))), 0.3)
            path = os.path.join(td, "x.coo")
            rk.save_tensor(xs, path)
            d["coo_dense"] = xs.to_dense().slices
            d["coo_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        d["meta"] = meta
        np.savez_compressed(os.path.join(HERE, "io_bytes.npz"), **d)
        print("wrote io_bytes")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        extra_cases(sys.argv[1:])
    else:
        main()
