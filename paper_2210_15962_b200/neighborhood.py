"""Incremental neighbourhood evaluation (drop-in for skewsaw.neighborhood,
neighborhood.py:1-100), on the device.

``EvalState`` / ``naive_oracle`` / ``flip`` / ``compute_deltas`` /
``apply_flip`` keep the reference's names, validation and results; the
delta and move arithmetic runs in the batched kernels of
csrc/neighborhood.cuh (sk_all_neighbor_deltas / sk_apply_neighbor).
``NeighborhoodBatch`` keeps S states resident on the device for large
sweeps (the reference handles one state per Python call).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _kernels, _lib
from .core import as_spins, autocorrelations, energy, expand_skew

__all__ = ["EvalState", "flip", "naive_oracle", "compute_deltas", "apply_flip", "NeighborhoodBatch"]


@dataclass(frozen=True)
class EvalState:
    """A pivot with its expansion, sidelobe array (entry L-k-1 holds C_k, as
    in the reference) and energy."""

    half: np.ndarray
    full: np.ndarray
    sidelobes: np.ndarray
    E: int

    @property
    def D(self) -> int:
        return self.half.size

    @property
    def L(self) -> int:
        return self.full.size


def _sidelobe_array(full: np.ndarray) -> np.ndarray:
    c = autocorrelations(full)  # c[k] = C_k
    return np.ascontiguousarray(c[::-1])


def naive_oracle(half) -> EvalState:
    """EvalState by full expansion and O(L^2) recomputation."""
    h = as_spins(half)
    full = expand_skew(h)
    return EvalState(half=h, full=full, sidelobes=_sidelobe_array(full), E=energy(full).E)


def flip(half, j: int) -> np.ndarray:
    h = as_spins(half)
    if not 0 <= j < h.size:
        raise ValueError(f"flip index {j} out of range for D={h.size}")
    out = h.copy()
    out[j] = -out[j]
    return out


def compute_deltas(state: EvalState) -> np.ndarray:
    """E(neighbour j) - E(pivot) for every j, from the sidelobes alone."""
    c = np.ascontiguousarray(state.sidelobes[::-1], dtype=np.int64)
    out = np.empty(state.D, dtype=np.int64)
    _kernels.all_neighbor_deltas(np.ascontiguousarray(state.full, dtype=np.int64), c, out)
    return out


def apply_flip(state: EvalState, j: int, deltas: np.ndarray) -> EvalState:
    """State of neighbour j, sidelobes updated incrementally."""
    if not 0 <= j < state.D:
        raise ValueError(f"flip index {j} out of range for D={state.D}")
    full = np.array(state.full, dtype=np.int64)
    c = np.ascontiguousarray(state.sidelobes[::-1], dtype=np.int64)
    _kernels.apply_neighbor(full, c, j)
    return EvalState(half=full[: state.D].copy(), full=full, sidelobes=c[::-1].copy(),
                     E=state.E + int(deltas[j]))


class NeighborhoodBatch:
    """S states of one length resident on the current CUDA device.

    Arrays use the reference's layout (full int64[S, L]; c int64[S, L] with
    c[:, k] = C_k; energies int64[S]).  ``deltas()`` evaluates every
    neighbourhood in one launch; ``apply(h)`` moves every state (h int64[S])
    in one launch and updates the energies from the last deltas."""

    def __init__(self, halves):
        import torch

        self.torch = torch
        halves = np.asarray(halves, dtype=np.int64)
        if halves.ndim != 2:
            raise ValueError("halves must be a 2-D array [S, D]")
        states = [naive_oracle(h) for h in halves]
        self.S, self.D = halves.shape
        self.L = 2 * self.D - 1
        dev = torch.device("cuda", torch.cuda.current_device())
        self.full = torch.from_numpy(np.stack([s.full for s in states])).to(dev)
        self.c = torch.from_numpy(np.stack([np.ascontiguousarray(s.sidelobes[::-1]) for s in states])).to(dev)
        self.E = torch.tensor([s.E for s in states], dtype=torch.int64, device=dev)
        self._d = torch.empty((self.S, self.D), dtype=torch.int64, device=dev)
        self._fresh = False

    def _stream(self):
        return self.torch.cuda.current_stream().cuda_stream

    def deltas(self):
        """Device tensor int64[S, D] of the current neighbourhoods."""
        _lib.check(_lib.load().sk_all_neighbor_deltas(self.L, self.S, self.full.data_ptr(), self.c.data_ptr(),
                                                      self._d.data_ptr(), self._stream()))
        self._fresh = True
        return self._d

    def apply(self, h):
        torch = self.torch
        ht = torch.as_tensor(np.asarray(h, dtype=np.int64).reshape(self.S)).to(self.full.device)
        if bool(((ht < 0) | (ht >= self.D)).any()):
            raise ValueError(f"flip index out of range for D={self.D}")
        if not self._fresh:
            self.deltas()
        self.E += self._d.gather(1, ht[:, None])[:, 0]
        _lib.check(_lib.load().sk_apply_neighbor(self.L, self.S, self.full.data_ptr(), self.c.data_ptr(),
                                                 ht.data_ptr(), self._stream()))
        self._fresh = False

    def halves(self) -> np.ndarray:
        return self.full[:, : self.D].cpu().numpy()

    def sidelobes(self) -> np.ndarray:
        """Reference layout: entry L-k-1 holds C_k."""
        return self.c.flip(1).cpu().numpy()
