"""CPU coverage of the N>1 path (gloo, world size 2 and 4).

Each rank runs, in fp64 numpy, the exact per-iteration schedule the CUDA grid
path executes (librescal_b200.so, rk_grid_init / enqueue_iteration with
p_r x p_c > 1):

  AllGather(row) / AllGather(col) of the owned A pieces
  local P = X_blk A_col, Q = X_blk^T A_row
  AllReduce(world) of [G = sum_pieces A_own^T A_own, S_t = A_row^T P_t]
  replicated core update, M = sum_t R^T G R + R G R^T
  ReduceScatter(row) of sum_t P R^T, ReduceScatter(col) of sum_t Q R
  own-piece A update

using the product's own block geometry (multigpu.piece_layout / block_of),
and checks the gathered factors against the serial oracle (the reference
requires <= 1e-8 for its own p=4 grid, test_dist_rescal.py:40-47).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2202_09512_b200.multigpu import block_of, grid_shape, piece_layout


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, n, m, k, iters, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pr, pc = grid_shape(world)
        gi, gj = rank // pc, rank % pc
        info = piece_layout(n, pr, pc, gi, gj)
        b = info["piece"]
        row_groups = [dist.new_group([i * pc + j for j in range(pc)]) for i in range(pr)]
        col_groups = [dist.new_group([i * pc + j for i in range(pr)]) for j in range(pc)]
        rowg, colg = row_groups[gi], col_groups[gj]

        x = np.random.default_rng(3).random((m, n, n))
        a0, r0 = oracle.random_init(n, k, m, 4)
        xb = block_of(x, n, info)                      # (m, pc*b, pr*b)
        pad = np.zeros((pr * pc * b, k))
        pad[:n] = a0
        own = pad[(gi * pc + gj) * b:(gi * pc + gj + 1) * b].copy()
        r = r0.copy()
        eps = 1e-16

        def allgather(piece, group, size):
            parts = [torch.zeros_like(torch.from_numpy(piece)) for _ in range(size)]
            dist.all_gather(parts, torch.from_numpy(piece), group=group)
            return np.concatenate([p.numpy() for p in parts], axis=0)

        def reduce_scatter(buf, group, size, idx):
            t = torch.from_numpy(np.ascontiguousarray(buf))
            dist.all_reduce(t, group=group)   # gloo has no reduce_scatter: same result
            return t.numpy()[idx * b:(idx + 1) * b]

        for _ in range(iters):
            arow = allgather(own, rowg, pc)    # pieces gi*pc + 0..pc-1
            acol = allgather(own, colg, pr)    # pieces 0..pr-1 * pc + gj
            p_loc = np.einsum("tij,jc->tic", xb, acol)
            q_loc = np.einsum("tij,ic->tjc", xb, arow)
            gs = np.concatenate([(own.T @ own)[None], np.einsum("ic,tid->tcd", arow, p_loc)], axis=0)
            t_gs = torch.from_numpy(gs)
            dist.all_reduce(t_gs)
            g, s = t_gs.numpy()[0], t_gs.numpy()[1:]
            for t in range(m):
                r[t] = r[t] * s[t] / (g @ (r[t] @ g) + eps)
            mm = sum(r[t].T @ g @ r[t] + r[t] @ g @ r[t].T for t in range(m))
            ui = sum(p_loc[t] @ r[t].T for t in range(m))
            uj = sum(q_loc[t] @ r[t] for t in range(m))
            num = reduce_scatter(ui, rowg, pc, gj) + reduce_scatter(uj, colg, pr, gi)
            own = own * num / (own @ mm + m * eps)
        full = allgather(own, dist.group.WORLD, world)
        # rank order is (gi, gj) row-major == piece order
        out_q.put((rank, full[:n], r))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 13), (4, 10), (8, 21)])
def test_grid_schedule_matches_serial_oracle(world, n):
    m, k, iters = 2, 3, 25
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, n, m, k, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = np.random.default_rng(3).random((m, n, n))
    a0, r0 = oracle.random_init(n, k, m, 4)
    a_ref, r_ref, _ = oracle.solve([x[t] for t in range(m)], k,
                                   oracle.OracleConfig(max_iters=iters, track_error=False), initial=(a0, r0))
    r_bytes = {rr.tobytes() for _, _, rr in res}
    assert len(r_bytes) == 1  # cores replicated byte-identically (test_dist_rescal.py:65-78)
    for _, a, rr in res:
        assert np.max(np.abs(a - a_ref) / np.maximum(np.abs(a_ref), 1e-300)) <= 1e-8
        assert np.max(np.abs(rr - r_ref) / np.maximum(np.abs(r_ref), 1e-300)) <= 1e-8
