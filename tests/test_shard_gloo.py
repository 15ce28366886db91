"""Multi-rank row-band orchestration (halo exchange, column-total exclusive scan)
on CPU with the gloo backend, world sizes 2 and 3.  Local compute is the oracle
(a numpy backend defined here), so this covers the host logic of shard.py; the
CUDA backend runs the same code path on GPUs."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

from conftest import REPO


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class NumpyBackend:
    def window(self, x, kind, w, stride, stats, pipeline="auto"):
        import torch

        from oracle import satsweep_oracle as O

        a = x.numpy()
        if a.dtype == np.int16:
            a = a.view(np.uint16)
        out = {}
        for s in stats:
            r = O.swa(a, w, s.value, stride)
            out[s] = torch.from_numpy(r.view(np.int64) if r.dtype == np.uint64 else r)
        return out

    def window_start(self, x, kind, w, stats):
        return self.window(x, kind, w, 1, stats)

    def window_finish(self, handle):
        return handle

    def band_totals(self, x, kind, squared):
        import torch

        from oracle import satsweep_oracle as O

        a = x.numpy()
        t = O.build_table(a, squared)
        last = t[-1].astype(np.uint64) if t.dtype != np.float64 else t[-1]
        tot = torch.from_numpy(last.view(np.int64) if last.dtype == np.uint64 else last.copy())
        return {"tot": None if squared else tot, "tot_sq": tot if squared else None, "x": a}

    def carry(self, gathered, rank):
        import torch

        g = gathered.numpy()
        if g.dtype == np.float64:
            return torch.from_numpy(g[:rank].sum(axis=0))
        return torch.from_numpy(g.view(np.uint64)[:rank].sum(axis=0, dtype=np.uint64).view(np.int64))

    def finish(self, x, kind, state, carry, carry_sq, squared):
        import torch

        from oracle import satsweep_oracle as O

        t = O.build_table(state["x"], squared)
        c = carry_sq if squared else carry
        if t.dtype == np.float64:
            if c is not None:
                t = t + c.numpy()[None, :]
            return torch.from_numpy(t), t.shape[1]
        t = t.astype(np.uint64)
        if c is not None:
            t = t + c.numpy().view(np.uint64)[None, :]
        return torch.from_numpy(t.view(np.int64)), t.shape[1]


def _worker(rank, world, port, img, w, stride, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "tests"))
    import torch
    import torch.distributed as dist

    from paper_2410_16291_b200 import shard
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows, cols = img.shape
        kind = ElemKind.from_dtype(img.dtype)
        a, b = shard.window_input_bands(rows, w, stride, world)[rank]
        res = shard.swa_sharded(torch.from_numpy(img[a:b].copy()), rows, cols, kind, w,
                                (StatKind.SUM, StatKind.MEAN), stride, backend=NumpyBackend())
        win = {k.value: v.numpy() for k, v in res.values.items()}
        # zero-copy layout: halo received in place into the band's storage
        storage, view = shard.band_storage(rows, cols, w, stride, torch.from_numpy(img).dtype)
        a, b = shard.window_input_bands(rows, w, stride, world)[rank]
        view.copy_(torch.from_numpy(img[a:b]))
        res2 = shard.swa_sharded(view, rows, cols, kind, w, (StatKind.SUM, StatKind.MEAN), stride,
                                 backend=NumpyBackend(), storage=storage)
        for k, v in res2.values.items():
            assert np.array_equal(v.numpy(), win[k.value]), k
        a, b = shard.table_input_bands(rows, world)[rank]
        tab = shard.build_sat_sharded(torch.from_numpy(img[a:b].copy()), rows, cols, kind, backend=NumpyBackend())
        # the combined step (bench.py at N > 1): windows of the output band and
        # global table rows of the OWNED window band, in one call
        comb = None
        if stride == 1:
            a, b = shard.window_input_bands(rows, w, 1, world)[rank]
            wr, tr = shard.swa_table_sharded(torch.from_numpy(img[a:b].copy()), rows, cols, kind, w,
                                             (StatKind.SUM,), backend=NumpyBackend())
            comb = (wr.rows, {k.value: v.numpy() for k, v in wr.values.items()}, tr.rows,
                    tr.values["table"].numpy())
        q.put((rank, res.rows, win, tab.rows, tab.values["table"].numpy(), comb))
    finally:
        dist.destroy_process_group()


def run(world, img, w, stride):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, img, w, stride, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda r: r[0])


@pytest.mark.parametrize("world,shape,w,stride",
                         [(2, (61, 37), 9, 1), (3, (50, 23), 17, 2), (2, (12, 40), 11, 1), (3, (12, 40), 11, 1)])
def test_sharded_matches_whole_image(world, shape, w, stride):
    from oracle import satsweep_oracle as O

    rng = np.random.default_rng(world * 100 + w)
    img = rng.integers(0, 256, size=shape, dtype=np.uint8)
    parts = run(world, img, w, stride)
    # window path: concatenated output bands == whole-image result
    sums = np.concatenate([p[2]["sum"] for p in parts if p[2]], axis=0).view(np.uint64)
    means = np.concatenate([p[2]["mean"] for p in parts if p[2]], axis=0)
    np.testing.assert_array_equal(sums, O.swa(img, w, "sum", stride))
    np.testing.assert_array_equal(means, O.swa(img, w, "mean", stride))
    # table path: rank g holds global table rows [a_g, a_{g+1}]
    full = O.build_table(img)
    for rank, _, _, (a, b), table, _ in parts:
        np.testing.assert_array_equal(table.view(np.uint64), full[a:b + 1])
    if stride == 1:
        combs = [p[5] for p in parts]
        sums2 = np.concatenate([c[1]["sum"] for c in combs if c[1]], axis=0).view(np.uint64)
        np.testing.assert_array_equal(sums2, O.swa(img, w, "sum"))
        assert combs[0][2][0] == 0 and combs[-1][2][1] == img.shape[0]
        for (_, _, (a, b), table) in combs:
            np.testing.assert_array_equal(table.view(np.uint64)[:, : img.shape[1] + 1], full[a:b + 1])


def test_geometry_helpers():
    from paper_2410_16291_b200 import shard

    for rows, w, s, n in [(100, 7, 1, 4), (100, 30, 3, 8), (9, 9, 1, 3), (70000, 256, 1, 8)]:
        owned = shard.window_input_bands(rows, w, s, n)
        assert owned[0][0] == 0 and owned[-1][1] == rows
        assert all(x[1] == y[0] for x, y in zip(owned, owned[1:]))
        need = shard.window_needed_rows(rows, w, s, n)
        out_r = (rows - w) // s + 1
        bands = shard.output_partition(out_r, n)
        for (lo, hi), (a, b) in zip(bands, need):
            if hi > lo:
                assert b - a == (hi - lo - 1) * s + w
    # C5 on 8 GPUs: halo of w-1 rows per boundary
    need = shard.window_needed_rows(70000, 256, 1, 8)
    owned = shard.window_input_bands(70000, 256, 1, 8)
    assert all(nb - ob == 255 for (na, nb), (oa, ob) in zip(need[:-1], owned[:-1]))
