"""List-sharded multi-GPU search: one process per GPU.

Every rank owns a subset of the inverted lists (and their coarse centroids)
and searches the WHOLE query batch:

  1. K1 over the owned centroids -> per query the nprobe smallest
     (d2, global cluster id) keys;
  2. all-gather of those keys, merge -> the global probe set, identical on
     every rank and identical to the 1-GPU selection (keys are a total order,
     d2 does not depend on the shard);
  3. K2-K4 over the owned probed lists -> local top-k keys per query, plus the
     global candidate count (from the replicated list lengths);
  4. all-gather of the top-k keys, merge, finalize -> ids / dists / short,
     bit-identical to the single-GPU result.

The orchestration is written against an `ops` object so that the exact same
protocol code runs with the CUDA ops (`CudaShardOps`) on the GPU box and with
injected CPU ops in the world-size-2 gloo tests.
"""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["shard_lists", "probe_frequency", "sharded_search", "CudaShardOps"]


def shard_lists(list_len: np.ndarray, s: int, world: int, probe_freq: np.ndarray | None = None) -> list[np.ndarray]:
    """Greedy largest-first partition of lists balanced over `world` ranks.
    Load of list c = its code bytes L_c * s, times its probe frequency when
    `probe_freq` is given (the scan work a rank gets is the code bytes of its
    lists weighted by how often they are probed).  Deterministic: ties by
    lower list id, then lower rank.  Returns the sorted list ids per rank."""
    list_len = np.asarray(list_len, dtype=np.int64)
    w = list_len.astype(np.float64) * s
    if probe_freq is not None:
        w = w * np.asarray(probe_freq, dtype=np.float64)
    w = w + 1.0
    order = np.lexsort((np.arange(list_len.size), -w))
    load = np.zeros(world, dtype=np.float64)
    owner = np.empty(list_len.size, dtype=np.int64)
    for c in order:
        r = int(np.argmin(load))  # first minimum -> lowest rank on ties
        owner[c] = r
        load[r] += w[c]
    return [np.flatnonzero(owner == r).astype(np.int32) for r in range(world)]


def probe_frequency(idx, sample: np.ndarray, nprobe: int) -> np.ndarray:
    """How often each list is probed by `sample` (e.g. base rows, which
    follow the query distribution) under the product's K1 -> counts [nlist]."""
    from .index import device_index
    sample = np.ascontiguousarray(sample, dtype=np.float32)
    probes = np.empty((sample.shape[0], nprobe), dtype=np.int64)
    h = device_index(idx)
    _lib.check(_lib.lib.ivfpq_select_clusters(h.handle, sample.ctypes.data, sample.shape[0], nprobe,
                                              probes.ctypes.data))
    return np.bincount(probes.ravel(), minlength=idx.nlist).astype(np.float64)


def sharded_search(ops, queries, k: int, nprobe: int, precision: str, all_gather):
    """Run the 4-step protocol.  `all_gather(t) -> stacked [world, ...]`.

    ops.select(queries, nprobe) -> keys [nq, nprobe] (uint64 / int64 view)
    ops.merge(stacked [W, nq, n], n_out) -> keys [nq, n_out]
    ops.scan(queries, probe_keys, nprobe, k, precision) -> (keys [nq, k], ncand [nq])
    ops.finalize(keys, ncand, k) -> (ids, dists, short)
    """
    local = ops.select(queries, nprobe)
    probes = ops.merge(all_gather(local), nprobe)
    keys, ncand = ops.scan(queries, probes, nprobe, k, precision)
    merged = ops.merge(all_gather(keys), k)
    return ops.finalize(merged, ncand, k)


class CudaShardOps:
    """The protocol's ops on one GPU shard, on torch CUDA tensors (uint64 keys
    are carried as int64 tensors; NCCL moves the bits unchanged)."""

    def __init__(self, dev_index, stream=None):
        import torch

        self.torch = torch
        self.dev = dev_index
        self.stream = stream

    def _st(self):
        return self.stream if self.stream is not None else self.torch.cuda.current_stream().cuda_stream

    def select(self, q, nprobe):
        out = self.torch.empty((q.shape[0], nprobe), dtype=self.torch.int64, device=q.device)
        _lib.check(_lib.lib.ivfpq_select_device(self.dev.handle, q.data_ptr(), q.shape[0], nprobe, out.data_ptr(),
                                                self._st()))
        return out

    def merge(self, stacked, n_out):
        W, nq, n_in = stacked.shape
        out = self.torch.empty((nq, n_out), dtype=self.torch.int64, device=stacked.device)
        _lib.check(_lib.lib.ivfpq_merge_keys_device(stacked.data_ptr(), W, nq, n_in, n_out, out.data_ptr(),
                                                    self._st()))
        return out

    def scan(self, q, probes, nprobe, k, precision):
        keys = self.torch.empty((q.shape[0], k), dtype=self.torch.int64, device=q.device)
        ncand = self.torch.empty(q.shape[0], dtype=self.torch.int64, device=q.device)
        _lib.check(_lib.lib.ivfpq_scan_device(self.dev.handle, q.data_ptr(), q.shape[0], probes.data_ptr(), nprobe,
                                              k, _lib.LUT_CODES[precision], keys.data_ptr(), ncand.data_ptr(),
                                              self._st()))
        return keys, ncand

    def finalize(self, keys, ncand, k):
        nq = keys.shape[0]
        ids = self.torch.empty((nq, k), dtype=self.torch.int64, device=keys.device)
        dists = self.torch.empty((nq, k), dtype=self.torch.float32, device=keys.device)
        short = self.torch.empty(nq, dtype=self.torch.int32, device=keys.device)
        _lib.check(_lib.lib.ivfpq_finalize_device(keys.data_ptr(), ncand.data_ptr(), nq, k, ids.data_ptr(),
                                                  dists.data_ptr(), short.data_ptr(), self._st()))
        return ids, dists, short


def torch_all_gather(group=None):
    """all_gather over torch.distributed returning a stacked tensor."""
    import torch
    import torch.distributed as dist

    def gather(t):
        W = dist.get_world_size(group)
        t = t.contiguous()
        if dist.get_backend(group) == "nccl":
            out = torch.empty((W,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t, group=group)
            return out
        parts = [torch.empty_like(t) for _ in range(W)]
        dist.all_gather(parts, t, group=group)
        return torch.stack(parts)

    return gather
