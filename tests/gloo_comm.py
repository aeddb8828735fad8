"""Test double of multi.NcclComm over torch.distributed gloo (host collectives).

The product's data plane is NCCL inside libtk_b200.so; NCCL cannot put two ranks on one GPU or
run without one, so the multi-rank host logic is checked on CPU (and the peer-store merge with
two processes sharing the single GPU of the test box) through this stand-in with the same
interface.  Test infrastructure only -- bench.py's one-GPU path check borrows it too."""

import torch
import torch.distributed as dist


class GlooComm:
    def __init__(self):
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self._pending = {}
        self._next = 0

    def counts_start(self, count, stream=None):
        t = torch.tensor([int(count)], dtype=torch.int64)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        work = dist.all_gather(out, t, async_op=True)
        self._next += 1
        self._pending[self._next] = (work, out)
        return self._next

    def counts_wait(self, ticket):
        work, out = self._pending.pop(ticket)
        work.wait()
        return [int(v.item()) for v in out]

    def allgather_counts(self, count, stream=None):
        return self.counts_wait(self.counts_start(count, stream))

    def gather_rows(self, subs, vals, counts, root=0, stream=None):
        nk = subs.shape[1] if subs.dim() == 2 else 1
        dev = subs.device
        s, v = subs.cpu(), vals.cpu()
        if self.rank == root:
            total = sum(counts)
            all_s = torch.empty((total, nk), dtype=subs.dtype)
            all_v = torch.empty(total, dtype=vals.dtype)
            off = 0
            for r in range(self.world):
                n = counts[r]
                if r == root:
                    all_s[off:off + n].copy_(s[:n])
                    all_v[off:off + n].copy_(v[:n])
                elif n:
                    dist.recv(all_s[off:off + n], src=r)
                    dist.recv(all_v[off:off + n], src=r)
                off += n
            return all_s.to(dev), all_v.to(dev)
        if counts[self.rank]:
            dist.send(s[:counts[self.rank]].contiguous(), dst=root)
            dist.send(v[:counts[self.rank]].contiguous(), dst=root)
        return None, None

    def allgather_bytes(self, data):
        out = [None] * self.world
        dist.all_gather_object(out, bytes(data))
        return out

    def barrier(self, stream=None):
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        dist.barrier()

    def allreduce_sum_(self, t, stream=None):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM)
        t.copy_(h)
        return t

    def close(self):
        pass
