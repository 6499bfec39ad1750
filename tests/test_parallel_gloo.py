"""World-size-2 gloo test of the list-sharded search protocol
(paper_2301_06672_b200/parallel.py): sharding, the two all-gathers and the
key merges must reproduce the single-process reference result bit for bit.
The per-shard compute is injected as CPU oracle ops (no GPU here); the
protocol code under test is the product's."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_case

EMPTY = np.uint64(0xFFFFFFFFFFFFFFFF)


class OracleShardOps:
    def __init__(self, c, owned):
        from oracle import ivfpq_np as onp
        self.onp = onp
        self.c = c
        self.owned = set(int(x) for x in owned)
        self.owned_arr = np.asarray(sorted(self.owned), dtype=np.int64)
        self.lens = np.diff(c["list_off"])
        self.s = c["centers"].shape[0]

    @staticmethod
    def _keys(d, ids):
        return (d.astype(np.float32).view(np.uint32).astype(np.uint64) << np.uint64(32)) | ids.astype(np.uint64)

    @staticmethod
    def _top(keys, n):
        keys = np.sort(keys[keys != EMPTY])[:n]
        return np.concatenate([keys, np.full(n - keys.size, EMPTY, np.uint64)])

    def select(self, q, nprobe):
        q = q.numpy()
        out = np.empty((q.shape[0], nprobe), np.uint64)
        for i in range(q.shape[0]):
            d2 = self.onp.squared_l2_to_all(self.c["coarse"][self.owned_arr], q[i])
            out[i] = self._top(self._keys(d2, self.owned_arr), nprobe)
        return torch.from_numpy(out.view(np.int64))

    def merge(self, stacked, n_out):
        st = stacked.numpy().view(np.uint64)
        W, nq, n_in = st.shape
        out = np.empty((nq, n_out), np.uint64)
        for i in range(nq):
            out[i] = self._top(st[:, i, :].reshape(-1), n_out)
        return torch.from_numpy(out.view(np.int64))

    def scan(self, q, probes, nprobe, k, prec):
        q = q.numpy()
        pr = probes.numpy().view(np.uint64)
        keys = np.empty((q.shape[0], k), np.uint64)
        ncand = np.zeros(q.shape[0], np.int64)
        off, ids, codes = self.c["list_off"], self.c["ids"], self.c["codes"]
        for i in range(q.shape[0]):
            parts = []
            for key in pr[i]:
                g = int(key & np.uint64(0xFFFFFFFF))
                ncand[i] += self.lens[g]
                if g not in self.owned or self.lens[g] == 0:
                    continue
                lut = self.onp.build_lut(self.c["centers"], q[i] - self.c["coarse"][g], prec)
                r = self.onp.scan_list(codes[off[g]:off[g + 1]].reshape(-1, self.s), lut, prec)
                parts.append(self._keys(r, ids[off[g]:off[g + 1]]))
            keys[i] = self._top(np.concatenate(parts) if parts else np.zeros(0, np.uint64), k)
        return torch.from_numpy(keys.view(np.int64)), torch.from_numpy(ncand)

    def finalize(self, keys, ncand, k):
        kk = keys.numpy().view(np.uint64)
        empty = kk == EMPTY
        ids = np.where(empty, -1, (kk & np.uint64(0xFFFFFFFF)).astype(np.int64))
        d = np.where(empty, np.float32(np.inf), (kk >> np.uint64(32)).astype(np.uint32).view(np.float32))
        return ids, d, (ncand.numpy() < k).astype(np.int32)


def _worker(rank, world, port, case, k, nprobe, prec, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from paper_2301_06672_b200 import parallel
    c = load_case(case)
    shards = parallel.shard_lists(np.diff(c["list_off"]), c["centers"].shape[0], world)
    ops = OracleShardOps(c, shards[rank])
    q = torch.from_numpy(c["queries"])
    ids, d, short = parallel.sharded_search(ops, q, k, nprobe, prec, parallel.torch_all_gather())
    np.savez(os.path.join(outdir, f"r{rank}.npz"), ids=ids, d=d, short=short)
    dist.destroy_process_group()


def test_shard_lists_balanced_and_partitioning():
    from paper_2301_06672_b200.parallel import shard_lists
    lens = np.random.default_rng(0).integers(0, 600, 1024)
    for world in (2, 4, 8):
        sh = shard_lists(lens, 64, world)
        allc = np.sort(np.concatenate(sh))
        assert np.array_equal(allc, np.arange(1024))
        loads = np.array([lens[s].sum() for s in sh])
        assert loads.max() - loads.min() <= lens.max()


@pytest.mark.parametrize("case,k,nprobe,prec", [("sift_mini", 10, 8, "e5m3"), ("small", 10, 4, "f16"),
                                                ("blobs", 20, 1, "f32")])
def test_two_rank_gloo_search_equals_single_process(tmp_path, case, k, nprobe, prec):
    from oracle import c_oracle
    world = 2
    port = 29500 + (abs(hash((case, k, nprobe, prec))) % 2000)
    mp.start_processes(_worker, args=(world, port, case, k, nprobe, prec, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    c = load_case(case)
    want_ids, want_d, want_short = c_oracle.search_batch(c["coarse"], c["centers"], c["list_off"], c["ids"],
                                                         c["codes"], c["queries"], k, nprobe, prec)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(z["ids"], want_ids)
        assert np.array_equal(z["d"], want_d)
        assert int(z["short"].sum()) == want_short
