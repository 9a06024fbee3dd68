"""Solver glue (Sec. 3.4): learning-rate schedules and the
divergence guard, with the iteration state in DEVICE memory (caffe_solver_state) so that a training
step captured once in a CUDA graph follows the schedule on every replay.

Argument marshalling only: lr_at_iter, the loss check and the update run in
libcaffe_b200.so (caffe_lr_at_iter, caffe_solver_begin / _end, caffe_sgd_update_solver).
"""
from __future__ import annotations

import ctypes

from . import _abi
from ._abi import call

POLICIES = {"fixed": _abi.CAFFE_LR_FIXED, "step": _abi.CAFFE_LR_STEP, "inv": _abi.CAFFE_LR_INV}


class DivergenceError(RuntimeError):
    """the loss of an iteration was not finite; that iteration changed no parameter."""


class Solver:
    def __init__(self, device, policy="fixed", base_lr=0.01, gamma=0.0, stepsize=1, power=0.0, momentum=0.9,
                 decay=5e-4):
        import torch
        self.torch = torch
        self.policy = _abi.LrPolicy(POLICIES[policy], float(base_lr), float(gamma), float(power), int(stepsize))
        self.momentum, self.decay = float(momentum), float(decay)
        assert ctypes.sizeof(_abi.SolverState) == 32
        self.state = torch.zeros(4, dtype=torch.int64, device=device)   # caffe_solver_state, zero = iteration 0

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def lr_at(self, it: int) -> float:
        v = ctypes.c_float()
        call("caffe_lr_at_iter", ctypes.byref(self.policy), int(it), ctypes.byref(v))
        return v.value

    def begin(self, loss=None):
        """After the step's loss: divergence check and this iteration's learning rate (on device)."""
        call("caffe_solver_begin", ctypes.byref(self.policy), ctypes.c_void_p(self.state.data_ptr()),
             ctypes.c_void_p(loss.data_ptr()) if loss is not None else None, self._stream())

    def end(self):
        call("caffe_solver_end", ctypes.c_void_p(self.state.data_ptr()), self._stream())

    def update(self, w, g, v, w_bf16=None, grad_scale=1.0):
        call("caffe_sgd_update_solver", ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(g.data_ptr()),
             ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(w_bf16.data_ptr()) if w_bf16 is not None else None,
             int(w.numel()), ctypes.c_void_p(self.state.data_ptr()), self.momentum, self.decay, float(grad_scale),
             self._stream())

    def read(self) -> dict:
        """Host copy of the device state (synchronises the current stream)."""
        raw = self.state.cpu().numpy().tobytes()
        st = _abi.SolverState.from_buffer_copy(raw)
        return {"iter": st.iter, "lr": st.lr, "diverged": bool(st.diverged), "diverged_iter": st.diverged_iter,
                "last_loss": st.last_loss}

    def check(self):
        s = self.read()
        if s["diverged"]:
            raise DivergenceError(f"non-finite loss at iteration {s['diverged_iter']} (S:524); "
                                  "the parameters keep their values from before that iteration")
        return s
