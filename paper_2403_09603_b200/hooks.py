"""Round-and-log attached to a PyTorch FP64 model (trainer side) -- the
caller of the path in BASELINE configs[3] and in the paper's PyTorch
implementation: every leaf module's forward output and every
module input gradient goes through the fused adaptive round-and-log
(``ops.round_and_log_adaptive``: per-tensor budget tau, device bisection,
sparse log), and the rounded FP64 grid values replace the originals, so
training proceeds on the b_r grid exactly as the reference trainer does
(protocol.py:259-285: forward stages, loss gradient, backward stages).

Nothing here synchronises with the host during the step: taus, counts and
logs stay on the device until ``collect()``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import ops


@dataclass
class HookRecord:
    name: str
    kind: str  # "fwd" | "bwd"
    numel: int
    budget: int
    pending: object  # ops.PendingAdaptive


@dataclass
class RoundAndLogHooks:
    model: torch.nn.Module
    b_r: int = 32
    budget_frac: float = 0.005
    iters: int = 30
    enabled: bool = True
    records: list[HookRecord] = field(default_factory=list)

    def __post_init__(self):
        self._handles = []
        for name, mod in self.model.named_modules():
            if any(True for _ in mod.children()):
                continue  # leaf modules only
            self._handles.append(mod.register_forward_hook(self._fwd_hook(name)))
            self._handles.append(mod.register_full_backward_hook(self._bwd_hook(name)))

    def _round(self, t: torch.Tensor, name: str, kind: str) -> torch.Tensor:
        if not (self.enabled and isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                and t.numel() > 0):
            return t
        n = t.numel()
        budget = int(self.budget_frac * n)
        d = t.detach()
        inplace = d.is_contiguous() and d.data_ptr() % 32 == 0
        flat = d.view(-1) if inplace else d.reshape(-1).clone()
        # in place: every tile's FP64 input is staged in shared memory before
        # its rounded values are stored back to the same addresses
        p = ops.round_and_log_adaptive(flat, self.b_r, budget, iters=self.iters, out_dtype=torch.float64,
                                       out=flat, check=False, tag=f"hooks_{kind}")
        self.records.append(HookRecord(name, kind, n, budget, p))
        return t if inplace else flat.view(t.shape)

    def _fwd_hook(self, name):
        def hook(mod, inp, out):
            if isinstance(out, torch.Tensor):
                y = self._round(out, name, "fwd")
                # out-of-place only for non-contiguous outputs: keep the module's graph
                return None if y is out else out + (y - out).detach()
            return None
        return hook

    def _bwd_hook(self, name):
        def hook(mod, grad_input, grad_output):
            if not any(isinstance(g, torch.Tensor) for g in grad_input):
                return None
            return tuple(self._round(g, name, "bwd") if isinstance(g, torch.Tensor) else g for g in grad_input)
        return hook

    def collect(self) -> dict:
        """Synchronise once: per-tensor taus and log sizes of the step."""
        taus, counts = [], []
        for r in self.records:
            _, log, tau = r.pending.finish()
            taus.append(tau)
            counts.append(log.count)
            assert log.count <= r.budget
        out = {"tensors": len(self.records), "elements": sum(r.numel for r in self.records),
               "logged": sum(counts), "fwd": sum(1 for r in self.records if r.kind == "fwd"),
               "bwd": sum(1 for r in self.records if r.kind == "bwd"),
               "tau_min": min(taus) if taus else None, "tau_max": max(taus) if taus else None}
        self.records.clear()
        return out

    def remove(self):
        for h in self._handles:
            h.remove()
        self._handles.clear()
