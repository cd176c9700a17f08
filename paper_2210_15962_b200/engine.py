"""Device-resident batch engine: the fast path behind ``runner.solve``.

One batch = W independent walks whose seeds are derived ON DEVICE from
(master_seed, batch, global walker index) -- runner.py:53-57 -- so no
per-walker host work exists (the reference spends ~2.4 us/walker in Python
deriving seeds and merging, runner.py:234-256).  Each device reduces its
walks to an ``sk_batch_summary`` (min over (E << 32 | walker), sum of steps,
winner's words); the host reads 80 bytes per device per batch.

Sharding: walkers [0, W) are split into contiguous slices, one per device
(in-process ``devices=[...]``) or per rank (``process_group``, one process per
GPU over NCCL).  Because seeds use the global walker index and the merge key
carries it, a batch's result is identical for any device count.  Across
ranks the exchange is one all_gather of every rank's summary [key, steps,
words] (a few dozen bytes per rank), merged on the host.

PyTorch is used only for device buffers, streams and torch.distributed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

SUMMARY_WORDS = _lib.SUMMARY_BYTES // 8  # 10 x uint64


@dataclass
class BatchResult:
    best_E: int
    walker: int           # global walker index of the winning walk
    steps_sum: int
    best_words: np.ndarray  # uint64[nw]


def _slices(W: int, parts: int):
    base, extra = divmod(W, parts)
    out, start = [], 0
    for i in range(parts):
        cnt = base + (1 if i < extra else 0)
        out.append((start, cnt))
        start += cnt
    return out


def decode_summary(raw: np.ndarray, nw: int) -> BatchResult | None:
    """uint64[10] summary -> BatchResult (None if the slice was empty)."""
    key = int(raw[0])
    if key == (1 << 64) - 1:
        return None
    steps = int(raw[1])
    return BatchResult(best_E=key >> 32, walker=key & 0xFFFFFFFF, steps_sum=steps,
                       best_words=raw[2:2 + nw].astype(np.uint64).copy())


def merge_across_ranks(win: BatchResult | None, steps: int, nw: int, process_group, device) -> BatchResult:
    """Merge per-rank batch results (one search); see merge_many_across_ranks."""
    return merge_many_across_ranks([win], [steps], nw, process_group, device)[0]


def merge_many_across_ranks(wins, steps, nw: int, process_group, device):
    """Merge per-rank results of R searches with ONE collective: every rank
    contributes its R summaries [key, steps, words...] (key = E << 32 |
    global walker, runner.py:252-256's rule as a MIN; an empty slice sends
    INT64_MAX) to an all_gather of R x (2 + nw) int64 words, then each rank
    merges on the host: lowest key wins, steps add up (runner.py:250-256)."""
    import torch
    import torch.distributed as dist

    R = len(wins)
    big = (1 << 63) - 1
    row = np.zeros((R, 2 + nw), dtype=np.int64)
    for r, (w, s) in enumerate(zip(wins, steps)):
        row[r, 0] = ((w.best_E << 32) | w.walker) if w is not None else big
        row[r, 1] = s
        if w is not None:
            row[r, 2:] = np.asarray(w.best_words, dtype=np.uint64).view(np.int64)
    world = dist.get_world_size(process_group)
    mine = torch.from_numpy(row).to(device)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=process_group)
    allr = np.stack([p.cpu().numpy() for p in parts])  # [world, R, 2 + nw]
    out = []
    for r in range(R):
        src = int(np.argmin(allr[:, r, 0]))
        key = int(allr[src, r, 0])
        if key == big:
            raise RuntimeError("no rank produced a walk for this batch")
        out.append(BatchResult(key >> 32, key & 0xFFFFFFFF, int(allr[:, r, 1].sum()),
                               allr[src, r, 2:].view(np.uint64).copy()))
    return out


class BatchEngine:
    """Runs batches of W walks of length n = walk_factor * D on GPU(s)."""

    def __init__(self, L: int, walkers: int, n: int, master_seed: int, devices=None, process_group=None):
        import torch

        self.torch = torch
        self.L = int(L)
        self.n = _lib.check_steps(n)
        self.D = (self.L + 1) // 2
        self.nw = (self.D + 63) // 64
        self.W = int(walkers)
        self.master = int(master_seed)
        self.pg = process_group
        lib = _lib.load()
        self.lib = lib
        if not torch.cuda.is_available():
            raise _lib.SokolError(_lib.SK_ERR_CUDA, "no CUDA device visible; the engine has no CPU path")
        if process_group is not None:
            import torch.distributed as dist

            self.rank = dist.get_rank(process_group)
            self.world = dist.get_world_size(process_group)
            devs = [torch.cuda.current_device()] if devices is None else list(devices)
            if len(devs) != 1:
                raise ValueError("with a process group each rank drives exactly one device")
            begin, cnt = _slices(self.W, self.world)[self.rank]
            self.parts = [(devs[0], begin, cnt)]
        else:
            self.rank, self.world = 0, 1
            devs = [torch.cuda.current_device()] if devices is None else list(devices)
            self.parts = [(d, b, c) for d, (b, c) in zip(devs, _slices(self.W, len(devs)))]
        self.streams = []
        self.summaries = []
        for dev, _, _ in self.parts:
            with torch.cuda.device(dev):
                self.streams.append(torch.cuda.Stream(device=dev))
                self.summaries.append(torch.empty(SUMMARY_WORDS, dtype=torch.int64, device=dev))
        self.host = torch.empty((len(self.parts), SUMMARY_WORDS), dtype=torch.int64, pin_memory=True)

    def launch(self, batch: int):
        """Enqueue batch `batch` on every local device (asynchronous)."""
        torch = self.torch
        for i, (dev, begin, cnt) in enumerate(self.parts):
            with torch.cuda.device(dev):
                st = self.streams[i]
                _lib.check(self.lib.sk_saw_batch(
                    self.L, self.n, None, self.master, int(batch), int(begin), int(cnt),
                    None, None, None, None, self.summaries[i].data_ptr(), st.cuda_stream,
                ))
                with torch.cuda.stream(st):
                    self.host[i].copy_(self.summaries[i], non_blocking=True)

    def collect(self) -> BatchResult:
        """Wait for the launched batch and merge it (across ranks if any)."""
        torch = self.torch
        for st in self.streams:
            st.synchronize()
        raw = self.host.numpy().view(np.uint64)
        local = [r for r in (decode_summary(raw[i], self.nw) for i in range(len(self.parts))) if r is not None]
        steps = sum(r.steps_sum for r in local)
        win = min(local, key=lambda r: (r.best_E, r.walker)) if local else None
        if self.pg is None:
            assert win is not None
            return BatchResult(win.best_E, win.walker, steps, win.best_words)
        return self._merge_ranks(win, steps)

    def _merge_ranks(self, win: BatchResult | None, steps: int) -> BatchResult:
        import torch.distributed as dist

        dev = self.parts[0][0]
        nccl = dist.get_backend(self.pg) == "nccl"
        tdev = self.torch.device("cuda", dev) if nccl else self.torch.device("cpu")
        return merge_across_ranks(win, steps, self.nw, self.pg, tdev)

    def run_batch(self, batch: int) -> BatchResult:
        self.launch(batch)
        return self.collect()

    # ---- R concurrent searches (sk_saw_multi) --------------------------------
    def run_multi(self, masters, batches) -> list[BatchResult]:
        """One batch of each of R independent searches (same L, W, n; own
        master seed and batch index) in one launch per device.  Result r is
        identical to BatchEngine(L, W, n, masters[r]).run_batch(batches[r])."""
        torch = self.torch
        R = len(masters)
        if R != len(batches) or R < 1:
            raise ValueError("masters and batches must be non-empty and of equal length")
        # pinned / device buffers, reused while they are large enough (capacity: a power of two)
        if getattr(self, "_multi_cap", 0) < R:
            cap = 1 << (R - 1).bit_length()
            self._multi_cap = cap
            self._multi_host = torch.empty(2 * cap, dtype=torch.int64, pin_memory=True)  # masters | batches
            self._multi_dev = []
            for dev, _, _ in self.parts:
                with torch.cuda.device(dev):
                    self._multi_dev.append((torch.empty(2 * cap, dtype=torch.int64, device=dev),
                                            torch.empty((cap, SUMMARY_WORDS), dtype=torch.int64, device=dev),
                                            torch.empty((cap, SUMMARY_WORDS), dtype=torch.int64, pin_memory=True)))
        mb = self._multi_host.numpy().view(np.uint64)
        mb[:R] = [int(m) & ((1 << 64) - 1) for m in masters]
        mb[R:2 * R] = [int(b) for b in batches]
        outs = []
        for i, (dev, begin, cnt) in enumerate(self.parts):
            d_in, summ, h = self._multi_dev[i]
            summ, h = summ[:R], h[:R]
            with torch.cuda.device(dev):
                st = self.streams[i]
                with torch.cuda.stream(st):
                    d_in[:2 * R].copy_(self._multi_host[:2 * R], non_blocking=True)
                _lib.check(self.lib.sk_saw_multi(
                    self.L, self.n, d_in.data_ptr(), d_in[R:].data_ptr(), R, int(begin), int(cnt),
                    summ.data_ptr(), st.cuda_stream,
                ))
                with torch.cuda.stream(st):
                    h.copy_(summ, non_blocking=True)
                outs.append((h,))
        for st in self.streams:
            st.synchronize()
        wins, steps = [], []
        for r in range(R):
            local = [x for x in (decode_summary(o[0][r].numpy().view(np.uint64), self.nw) for o in outs) if x is not None]
            steps.append(sum(x.steps_sum for x in local))
            wins.append(min(local, key=lambda x: (x.best_E, x.walker)) if local else None)
        if self.pg is None:
            return [BatchResult(w.best_E, w.walker, s, w.best_words) for w, s in zip(wins, steps)]
        import torch.distributed as dist

        dev = self.parts[0][0]
        tdev = torch.device("cuda", dev) if dist.get_backend(self.pg) == "nccl" else torch.device("cpu")
        return merge_many_across_ranks(wins, steps, self.nw, self.pg, tdev)
