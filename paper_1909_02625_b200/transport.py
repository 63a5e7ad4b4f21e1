"""Stage-to-stage packet transport between ranks (one process per GPU).

The reference's only concurrency boundary is ``_ThreadQueue.put/get``
(pipeline.py:176-205) inside one process; SPEC.md:362 names the queue as the
extension point for inter-machine transport. Here a cross-rank FIFO edge is
carried by point-to-point send/recv: NCCL over NVLink/NVSwitch on GPUs, gloo
for the CPU multi-process tests. Each message is (header, tensor); the header
carries the batch-index tag (and the labels for activations) so the consumer
re-checks the reference's gradient-meets-activation assertion.
"""

from __future__ import annotations


class LocalTransport:
    rank = 0
    world = 1

    def exchange(self, sends, recvs) -> None:
        if sends or recvs:
            raise RuntimeError("single-process transport cannot exchange packets")


class TorchDistTransport:
    """Batched isend/irecv over the default torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, sends, recvs) -> None:
        """sends: [(dst, header, tensor)], recvs: [(src, header_buf, tensor_buf)].

        Messages between one (src, dst) pair are matched in list order on both
        sides; the engine builds both lists edge by edge in ascending order."""
        dist = self.dist
        ops = []
        for dst, hdr, ten in sends:
            ops.append(dist.P2POp(dist.isend, hdr, dst, self.group))
            ops.append(dist.P2POp(dist.isend, ten, dst, self.group))
        for src, hdr, ten in recvs:
            ops.append(dist.P2POp(dist.irecv, hdr, src, self.group))
            ops.append(dist.P2POp(dist.irecv, ten, src, self.group))
        if not ops:
            return
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def default_transport():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return LocalTransport()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return TorchDistTransport()
    return LocalTransport()
