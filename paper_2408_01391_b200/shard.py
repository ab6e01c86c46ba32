"""Row-sharded multi-GPU Lloyd.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Each
rank owns a contiguous row shard of X and a replica of the centroids; the
only exchange per iteration is ONE packed all-reduce of
``[per-cluster float64 sums (K*D) | counts (K, as float64: exact below 2^53)
| partial inertia | changed-label count]`` (4.2 MB at K=4096, D=128) -- after
it every rank runs the identical finalize, so the centroids stay bit-identical
across ranks.  With the NCCL backend the pack, the all-reduce and the unpack
are captured in the step's CUDA graph (``capturable``): a sharded step is one
graph replay like a single-GPU step.  The rare empty-cluster reseed is a
MAXLOC: every rank offers its shard's farthest point, ties resolve to the
lowest global row index (np.argmax's first-maximum rule, kmeans.py:197-206).

Shards start on multiples of ``ALIGN`` rows, so the reference's logical
fault-tile grid (bm = 32 or 64 rows) maps onto shards without splitting a
tile, and every shard's tiles are the global tiles offset by
``row_offset // bm``.

Parity caveat: the float64 sums are summed per shard then across ranks, so
for world_size > 1 the summation association differs from the reference's
single ascending pass (centroids agree to ~1e-16 relative; labels are
row-local and exact given identical centroids).
"""

from __future__ import annotations

ALIGN = 256


class ShardComm:
    def __init__(self, row_offset, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.row_offset = int(row_offset)
        # NCCL collectives can be captured in a CUDA graph; gloo cannot
        self.capturable = dist.get_backend(group) == "nccl"
        self._buf = None

    @staticmethod
    def shard_bounds(n_rows, world, rank, align=ALIGN):
        """[lo, hi) of `rank`: near-equal shards whose starts are multiples of
        `align` rows (the last shard takes the remainder)."""
        per = -(-n_rows // world)
        per = -(-per // align) * align
        lo = min(n_rows, rank * per)
        return lo, min(n_rows, lo + per)

    def all_reduce_(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def reduce_partials(self, sums, counts, ctl_f64, ctl_i32, iteration=0):
        """sums (K, D) f64, counts (K,) i64, ctl_f64[0] = partial inertia,
        ctl_i32[0] = this shard's labels-unchanged flag; all in place.  No
        allocation after the first call (graph-capturable)."""
        import torch

        k, d = sums.shape
        n = k * d + k + 2
        if self._buf is None or self._buf.numel() != n or self._buf.device != sums.device:
            self._buf = torch.empty(n, dtype=torch.float64, device=sums.device)
        buf = self._buf
        kd = k * d
        buf[:kd].view(k, d).copy_(sums)
        buf[kd:kd + k].copy_(counts)
        buf[kd + k:kd + k + 1].copy_(ctl_f64[0:1])
        buf[kd + k + 1:].copy_(ctl_i32[0:1]).neg_().add_(1.0)  # changed = 1 - unchanged
        self.dist.all_reduce(buf, group=self.group)
        sums.copy_(buf[:kd].view(k, d))
        counts.copy_(buf[kd:kd + k])
        ctl_f64[0:1].copy_(buf[kd + k:kd + k + 1])
        ctl_i32[0:1].copy_(buf[kd + k + 1:].eq(0.0))

    def reseed(self, x_t, counts, sq, cent):
        """Empty clusters (ascending) take successive global farthest points."""
        import torch

        empty = torch.nonzero(counts <= 0).flatten().tolist()
        dev = x_t.device
        d = x_t.shape[1]
        for j in empty:
            if sq.numel():
                li = int(torch.argmax(sq).item())
                val = sq[li].to(torch.float64)
                row = x_t[li].to(torch.float64)
            else:
                li, val, row = -1, torch.tensor(float("-inf"), device=dev, dtype=torch.float64), \
                    torch.zeros(d, dtype=torch.float64, device=dev)
            gidx = self.row_offset + li if li >= 0 else 2 ** 62
            mine = torch.cat([val.reshape(1), torch.tensor([float(gidx)], dtype=torch.float64,
                                                           device=dev), row])
            got = [torch.empty_like(mine) for _ in range(self.world)]
            self.dist.all_gather(got, mine, group=self.group)
            best = None
            for r, g in enumerate(got):
                v, gi = float(g[0].item()), float(g[1].item())
                nan = v != v  # numpy argmax: NaN is the maximum, then max value, then min index
                key = (nan, 0.0 if nan else v, -gi)
                if best is None or key > best[0]:
                    best = (key, r, g)
            _, owner, g = best
            cent[j].copy_(g[2:].to(cent.dtype))
            if owner == self.rank and li >= 0:
                sq[li] = float("-inf")
