"""Round-and-log attached to a PyTorch FP64 model (trainer side) -- the
caller of the path in BASELINE configs[3] and in the paper's PyTorch
implementation: every leaf module's forward output and every
module input gradient goes through the fused adaptive round-and-log
(``ops.round_and_log_adaptive``: per-tensor budget tau, device bisection,
sparse log), and the rounded FP64 grid values replace the originals, so
training proceeds on the b_r grid exactly as the reference trainer does
(protocol.py:259-285: forward stages, loss gradient, backward stages).

``ReplayHooks`` is the auditor side (protocol._AuditorChannel.process,
protocol.py:212-216, on a torch model): the same hook points replay the
trainer's per-tensor logs in place (``ops.replay``), so an auditor whose
hardware computes slightly different FP64 values lands on the trainer's grid
values bit for bit.

Nothing here synchronises with the host during the step: taus, counts and
logs stay on the device until ``collect()``, which reads the whole step's
taus and counts in one copy.  Result slots (tau, error/count words) and log
buffers are reused from step to step, so a steady-state step allocates
nothing (a device allocation inside a step can stall the stream).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _device as D
from . import _lib
from . import ops


@dataclass
class HookRecord:
    name: str
    kind: str  # "fwd" | "bwd"
    numel: int
    budget: int
    pending: object  # ops.PendingAdaptive
    slot: int = 0    # row of the hooks' result arena


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
        self._flags = torch.zeros((0, 6), dtype=torch.int64, device="cuda")  # per call: err, -, counters
        self._taus = torch.zeros(0, dtype=torch.float64, device="cuda")
        self._logs: list[torch.Tensor] = []  # per call index: log buffer, reused while large enough
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
        k = len(self.records)
        if k >= self._flags.shape[0]:  # first steps only: grow the result slots
            grow = max(64, 2 * self._flags.shape[0])
            self._flags = torch.cat([self._flags, torch.zeros((grow, 6), dtype=torch.int64, device="cuda")])
            self._taus = torch.cat([self._taus, torch.zeros(grow, dtype=torch.float64, device="cuda")])
            for r in self.records:  # keep pending results pointing at live slots
                r.pending.flags = D.Flags(buf=self._flags[r.slot])
                r.pending.tau = self._taus[r.slot:r.slot + 1]
        if k >= len(self._logs):
            self._logs.append(torch.empty(0, dtype=torch.int64, device="cuda"))
        if self._logs[k].numel() < budget + 1:
            self._logs[k] = torch.empty(budget + 1, dtype=torch.int64, device="cuda")
        # in place: every tile's FP64 input is staged in shared memory before
        # its rounded values are stored back to the same addresses
        p = ops.round_and_log_adaptive(flat, self.b_r, budget, iters=self.iters, out_dtype=torch.float64,
                                       out=flat, log_out=self._logs[k][: budget + 1], check=False,
                                       tag=f"hooks_{kind}", tau_out=self._taus[k:k + 1], flags_out=self._flags[k])
        self.records.append(HookRecord(name, kind, n, budget, p, k))
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

    def loss_grad(self, output: torch.Tensor, name: str = "loss") -> torch.Tensor:
        """Route the loss gradient (d loss / d ``output``, the model's output)
        through the round-and-log as well -- protocol.py:277-280, where the
        reference passes the loss gradient through the channel before the
        backward stages.  Call on the output before ``backward()``; the
        gradient is rounded and logged when autograd reaches it (recorded
        with kind "loss")."""
        if self.enabled and isinstance(output, torch.Tensor) and output.requires_grad:
            output.register_hook(lambda g: self._round(g, name, "loss"))
        return output

    def collect(self, keep_logs: bool = False) -> dict:
        """Synchronise once: per-tensor taus and log sizes of the step (one
        copy of the step's result slots), then clear the slots for the next
        step.  Raises the reference's errors like PendingAdaptive.finish.
        keep_logs: also return the step's logs (``"logs"``: one (name, kind,
        int64 words) per hooked tensor, in call order, copied out of the
        reused buffers) -- what the trainer ships to an auditor."""
        m = len(self.records)
        fl = self._flags[:m].cpu().tolist()
        taus = self._taus[:m].cpu().tolist()
        records = list(self.records)
        self._flags[:m].zero_()  # the slots start the next step cleared, whatever is raised below
        self.records.clear()
        counts = []
        for r, f in zip(records, fl):
            D.raise_fpround(int(f[0]) & 0xFFFFFFFF)
            if f[2] > r.budget + 1:
                raise ops.LogOverflow(f"sparse log needs {f[2]} words, capacity {r.budget + 1}")
            counts.append(int(f[2]))
            assert f[2] <= r.budget
        out = {"tensors": m, "elements": sum(r.numel for r in records),
               "logged": sum(counts), "fwd": sum(1 for r in records if r.kind == "fwd"),
               "bwd": sum(1 for r in records if r.kind == "bwd"),
               "loss": sum(1 for r in records if r.kind == "loss"),
               "tau_min": min(taus) if taus else None, "tau_max": max(taus) if taus else None,
               "taus": taus, "counts": counts,
               "calls": [(r.name, r.kind, r.numel, r.budget) for r in records]}
        if keep_logs:
            out["logs"] = [(r.name, r.kind, self._logs[r.slot][:c].clone()) for r, c in zip(records, counts)]
        return out

    def remove(self):
        for h in self._handles:
            h.remove()
        self._handles.clear()


@dataclass
class ReplayHooks:
    """Auditor side: at the trainer's hook points, in the trainer's call
    order, round each tensor in place with the trainer's log forcing the
    logged directions (``ops.replay``: rev_array, fpround.py:227-247).
    ``logs`` is ``RoundAndLogHooks.collect(keep_logs=True)["logs"]`` of the
    step being audited.  ``perturb`` (optional, tensor -> None, in place)
    runs before each replay: a stand-in for the auditor's hardware computing
    slightly different values."""

    model: torch.nn.Module
    logs: list
    b_r: int = 32
    perturb: object = None
    enabled: bool = True

    def __post_init__(self):
        self._handles = []
        self._k = 0
        self._flags = torch.zeros((max(len(self.logs), 1), 6), dtype=torch.int64, device="cuda")
        for name, mod in self.model.named_modules():
            if any(True for _ in mod.children()):
                continue
            self._handles.append(mod.register_forward_hook(self._fwd_hook(name)))
            self._handles.append(mod.register_full_backward_hook(self._bwd_hook(name)))

    def _replay(self, t: torch.Tensor, name: str, kind: str) -> torch.Tensor:
        if not (self.enabled and isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                and t.numel() > 0):
            return t
        k = self._k
        if k >= len(self.logs) or self.logs[k][0] != name or self.logs[k][1] != kind:
            want = self.logs[k][:2] if k < len(self.logs) else None
            raise RuntimeError(f"audit out of step at hooked tensor {k}: trainer {want}, auditor {(name, kind)}")
        self._k += 1
        d = t.detach()
        inplace = d.is_contiguous() and d.data_ptr() % 32 == 0
        flat = d.view(-1) if inplace else d.reshape(-1).clone()
        if self.perturb is not None:
            self.perturb(flat)
        f = D.Flags(buf=self._flags[k])
        _lib_call_replay(flat, self.b_r, self.logs[k][2], f)
        return t if inplace else flat.view(t.shape)

    def _fwd_hook(self, name):
        def hook(mod, inp, out):
            if isinstance(out, torch.Tensor):
                y = self._replay(out, name, "fwd")
                return None if y is out else out + (y - out).detach()
            return None
        return hook

    def _bwd_hook(self, name):
        def hook(mod, grad_input, grad_output):
            if not any(isinstance(g, torch.Tensor) for g in grad_input):
                return None
            return tuple(self._replay(g, name, "bwd") if isinstance(g, torch.Tensor) else g for g in grad_input)
        return hook

    def loss_grad(self, output: torch.Tensor, name: str = "loss") -> torch.Tensor:
        """The auditor's side of ``RoundAndLogHooks.loss_grad``: the loss
        gradient is replayed against the trainer's log at the same point."""
        if self.enabled and isinstance(output, torch.Tensor) and output.requires_grad:
            output.register_hook(lambda g: self._replay(g, name, "loss"))
        return output

    def collect(self) -> dict:
        """Synchronise once: per-tensor corrections (elements where the log
        overrode plain rounding), errors raised as the reference does."""
        m = self._k
        fl = self._flags[:m].cpu().tolist()
        self._flags[:m].zero_()
        self._k = 0
        for f in fl:
            if int(f[0]) & _lib.ERR_BAD_SPARSE:
                raise ops.SparseLogError("sparse log is not strictly ascending")
            D.raise_fpround(int(f[0]) & 0xFFFFFFFF)
        if m != len(self.logs):
            raise RuntimeError(f"audit out of step: {m} hooked tensors, the trainer logged {len(self.logs)}")
        return {"tensors": m, "corrections": [int(f[2]) for f in fl]}

    def remove(self):
        for h in self._handles:
            h.remove()
        self._handles.clear()


@torch.no_grad()
def round_parameters(model: torch.nn.Module, b_r: int = 32) -> None:
    """Every FP64 parameter onto the b_r grid in place after the update, no
    log (protocol.py:286-293: ``stage.W = rnd_array(new_W, b_r)`` -- the
    stored parameters live on the grid).  One elementwise rounding launch per
    parameter; errors (non-finite / out of range) raise like rnd_array."""
    flags = D.Flags()
    launched = False
    for p in model.parameters():
        if not (p.is_cuda and p.dtype == torch.float64 and p.numel()):
            continue
        d = p.detach()
        inplace = d.is_contiguous() and d.data_ptr() % 32 == 0
        flat = d.view(-1) if inplace else d.reshape(-1).clone()
        _lib.call("vt_round_log", D.ptr(flat), flat.numel(), b_r, 0.0, _lib.OUT_F64, D.ptr(flat), None, 0, 0,
                  None, None, None, None, 0, None, flags.cnt_ptr, flags.err_ptr, None, 0, D.stream_ptr())
        if not inplace:
            d.copy_(flat.view(d.shape))
        launched = True
    if launched:
        D.raise_fpround(flags.read()[0])


def _lib_call_replay(flat: torch.Tensor, b_r: int, words: torch.Tensor, f) -> None:
    """In-place FP64 replay of one tensor against its sparse log (the fused
    replay stages each tile before writing it back)."""
    ws = D.workspace(int(_lib.lib().vt_replay_workspace(flat.numel())), "replay_hooks")
    w = words.contiguous()
    _lib.call("vt_replay", D.ptr(flat), flat.numel(), b_r, _lib.LOG_SPARSE, D.ptr(w), w.numel(), 0,
              _lib.OUT_F64, D.ptr(flat), f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
