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

import time
from collections import deque


class LocalTransport:
    rank = 0
    world = 1

    def exchange(self, sends, recvs, timeout_s=None) -> None:
        if sends or recvs:
            raise RuntimeError("single-process transport cannot exchange packets")

    def drain(self, timeout_s=None) -> None:
        pass


class TorchDistTransport:
    """Batched isend/irecv over the default torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._inflight = deque()  # NCCL: (issue time, requests) not yet known complete

    def exchange(self, sends, recvs, timeout_s: float | None = None) -> None:
        """sends: [(dst, header, tensor)], recvs: [(src, header_buf, tensor_buf)].

        Messages between one (src, dst) pair are matched in list order on both
        sides; the engine builds both lists edge by edge in ascending order.
        timeout_s: the watchdog (pipeline.py:644-657) -- raise TimeoutError if the
        requests have not completed by then (a stalled or dead peer)."""
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
        reqs = dist.batch_isend_irecv(ops)
        if timeout_s is None:
            for req in reqs:
                req.wait()
            return
        deadline = time.monotonic() + timeout_s
        if dist.get_backend(self.group) == "gloo":
            # gloo completes a request inside wait(); its timeout raises (RuntimeError "Timed out")
            from datetime import timedelta

            for i, req in enumerate(reqs):
                left = deadline - time.monotonic()
                try:
                    req.wait(timeout=timedelta(seconds=max(left, 1e-3)))
                except RuntimeError as exc:
                    if time.monotonic() < deadline and "imed out" not in str(exc):
                        raise
                    raise TimeoutError(f"{len(reqs) - i} of {len(reqs)} transfers pending after {timeout_s}s") from exc
            return
        # NCCL: wait() only orders the current stream after the transfer (the host goes on
        # enqueueing the next step); the watchdog retires completed batches as later steps are
        # issued and raises once a batch has been pending for timeout_s
        for req in reqs:
            req.wait()
        self._inflight.append((time.monotonic(), reqs))
        self._retire(timeout_s, block=False)

    def _retire(self, timeout_s, block: bool) -> None:
        while self._inflight:
            t0, reqs = self._inflight[0]
            if all(r.is_completed() for r in reqs):
                self._inflight.popleft()
                continue
            waited = time.monotonic() - t0
            if timeout_s is not None and waited > timeout_s:
                n = sum(1 for r in reqs if not r.is_completed())
                raise TimeoutError(f"{n} of {len(reqs)} transfers pending after {timeout_s}s")
            if not block:
                return
            time.sleep(2e-4)

    def drain(self, timeout_s=None) -> None:
        """Block until every issued transfer completed (sync points), under the watchdog."""
        self._retire(timeout_s, block=True)


def default_transport():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return LocalTransport()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return TorchDistTransport()
    return LocalTransport()
