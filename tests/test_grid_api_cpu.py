"""CPU coverage of the grid-facing drop-in names (no GPU).

* ``partition_block`` is the reference's own square-grid cut
  (tensor.py:339-362); ``grid_block`` / ``BlockSource`` cut the engine's
  p_r x p_c piece layout, from memory or from a memory-mapped RSK1 file, and
  must give exactly ``block_of`` of the whole tensor on every rank.
* ``gather_factors`` (dist_rescal.py:218-234) under gloo, world size 2 and 4:
  stacks the row sets of grid column 0 and rejects a core stack that differs
  between ranks with the reference's GridError text.
* ``KernelCounters`` keeps the reference's accounting interface (grid.py:72-94).
* Files: the writer produces the reference writer's exact bytes
  (tests/golden/io_bytes.npz, made by the reference's save_tensor /
  save_matrix) and the loader reads them back.
"""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2202_09512_b200 as rk
from conftest import golden
from paper_2202_09512_b200.multigpu import block_of, csr_block_of, grid_shape, piece_layout


def test_partition_block_is_the_reference_cut():
    x = np.random.default_rng(0).random((2, 7, 7))
    t = rk.RelTensor(x)
    for g in (1, 2, 3):
        b = rk.block_dim(7, g)
        for i in range(g):
            for j in range(g):
                blk = rk.partition_block(t, g, i, j)
                ref = np.zeros((2, b, b))
                r0, c0 = i * b, j * b
                sub = x[:, r0:min(r0 + b, 7), c0:min(c0 + b, 7)]
                ref[:, :sub.shape[1], :sub.shape[2]] = sub
                np.testing.assert_array_equal(blk.slices, ref)
                assert (blk.row_start, blk.col_start, blk.block_dim) == (r0, c0, b)
    with pytest.raises(rk.DataError, match="outside 2x2 grid"):
        rk.partition_block(t, 2, 2, 0)
    s = rk.SparseRelTensor([sp.csr_matrix(x[0] * (x[0] > 0.5)), sp.csr_matrix(x[1] * (x[1] > 0.5))])
    blk = rk.partition_block(s, 2, 1, 0)
    np.testing.assert_array_equal(blk.slices[0].toarray()[:3, :4], (x[0] * (x[0] > 0.5))[4:7, 0:4])


@pytest.mark.parametrize("n,p", [(10, 2), (13, 4), (17, 8)])
def test_grid_block_and_file_source_match_block_of(tmp_path, n, p):
    m = 3
    x = np.random.default_rng(n).random((m, n, n)).astype(np.float32)
    t = rk.RelTensor(x)
    path = tmp_path / "x.rsk"
    rk.save_tensor(t, str(path))
    src = rk.BlockSource.from_file(str(path))
    assert (src.n, src.m, src.dtype) == (n, m, np.float32)
    pr, pc = grid_shape(p)
    for r in range(p):
        lay = piece_layout(n, pr, pc, r // pc, r % pc)
        ref = block_of(x, n, lay)
        np.testing.assert_array_equal(src.block(lay), ref)
        np.testing.assert_array_equal(rk.grid_block(t, pr, pc, r // pc, r % pc).slices, ref)
    # the blocks partition X: the squares sum to ||X||^2
    tot = sum(float(np.sum(block_of(x, n, piece_layout(n, pr, pc, r // pc, r % pc)).astype(np.float64) ** 2))
              for r in range(p))
    assert abs(tot - float(np.sum(x.astype(np.float64) ** 2))) <= 1e-9 * tot


def test_sparse_grid_block_matches_dense_cut():
    n, m = 11, 2
    rng = np.random.default_rng(4)
    dense = rng.random((m, n, n)) * (rng.random((m, n, n)) < 0.3)
    s = rk.SparseRelTensor([sp.csr_matrix(dense[t]) for t in range(m)])
    for r in range(4):
        lay = piece_layout(n, 2, 2, r // 2, r % 2)
        blk = rk.grid_block(s, 2, 2, r // 2, r % 2)
        np.testing.assert_array_equal(np.stack([q.toarray() for q in blk.slices]), block_of(dense, n, lay))
        for q in csr_block_of(s.slices, n, lay):
            assert q.has_sorted_indices


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _gather_rank(rank, world, port, n, k, bad_rank, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pr, pc = grid_shape(world)
        lay = piece_layout(n, pr, pc, rank // pc, rank % pc)
        a = np.arange(n * k, dtype=np.float64).reshape(n, k) / 7.0
        pad = np.zeros((pr * pc * lay["piece"], k))
        pad[:n] = a
        r = np.full((2, k, k), 0.5)
        if rank == bad_rank:
            r[1, 0, 0] = np.nextafter(0.5, 1.0)
        rows = np.arange(lay["row0"], lay["row0"] + lay["rows"])
        df = rk.DistFactors(a_row=pad[rows], a_col=pad[lay["colmap"]], r=r, i=lay["gi"], j=lay["gj"], n_global=n)
        try:
            f = rk.gather_factors(df)
            out_q.put((rank, "ok", np.array_equal(f.A, a) and np.array_equal(f.R, r)))
        except rk.GridError as ex:
            out_q.put((rank, "err", str(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,bad", [(2, -1), (4, -1), (4, 2)])
def test_gather_factors_gloo(world, bad):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_rank, args=(r, world, port, 13, 3, bad, q)) for r in range(world)]
    for pr_ in procs:
        pr_.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr_ in procs:
        pr_.join(timeout=60)
        assert pr_.exitcode == 0
    if bad < 0:
        assert all(kind == "ok" and ok for _, kind, ok in res), res
    else:
        assert all(kind == "err" and msg == f"core stack differs on rank {bad}: broken run" for _, kind, msg in res)


def test_kernel_counters_interface():
    c = rk.KernelCounters()
    c.add_flops("gram_mul", 10)
    c.add_flops("gram_mul", 5)
    c.add_flops("matrix_mul", 7)
    with c.timed("matrix_mul"):
        pass
    assert c.flops == {"gram_mul": 15, "matrix_mul": 7} and c.total_flops() == 22
    assert c.seconds["matrix_mul"] >= 0.0


def test_files_are_byte_compatible_with_the_reference(tmp_path):
    g = golden("io_bytes")
    for tag in ("f32", "f64"):
        p = tmp_path / f"{tag}.rsk"
        rk.save_tensor(rk.RelTensor(g[f"dense_{tag}_X"]), str(p))
        assert p.read_bytes() == g[f"dense_{tag}_bytes"].tobytes()
        ref = tmp_path / f"ref_{tag}.rsk"
        ref.write_bytes(g[f"dense_{tag}_bytes"].tobytes())
        y = rk.load_tensor(str(ref))
        assert y.slices.dtype == g[f"dense_{tag}_X"].dtype
        np.testing.assert_array_equal(y.slices, g[f"dense_{tag}_X"])
    p = tmp_path / "a.rskm"
    rk.save_matrix(g["matrix_A"], str(p))
    assert p.read_bytes() == g["matrix_bytes"].tobytes()
    ref = tmp_path / "ref.rskm"
    ref.write_bytes(g["matrix_bytes"].tobytes())
    np.testing.assert_array_equal(rk.load_matrix(str(ref)), g["matrix_A"])
    xs = rk.SparseRelTensor([sp.csr_matrix(s) for s in g["coo_dense"]])
    p = tmp_path / "x.coo"
    rk.save_tensor(xs, str(p))
    assert p.read_bytes() == g["coo_bytes"].tobytes()


def test_dense_file_errors(tmp_path):
    p = tmp_path / "bad.rsk"
    p.write_bytes(b"RSKX" + bytes(21))
    with pytest.raises(rk.DataError, match="malformed header: bad magic"):
        rk.load_tensor(str(p), format="dense-binary")
    p.write_bytes(b"RSK1" + bytes(5))
    with pytest.raises(rk.DataError, match="malformed header: truncated"):
        rk.load_tensor(str(p))
    t = rk.RelTensor(np.ones((1, 3, 3), dtype=np.float32))
    rk.save_tensor(t, str(p))
    p.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(rk.DataError, match="dimension mismatch: expected 36 payload bytes, got 32"):
        rk.load_tensor(str(p))
