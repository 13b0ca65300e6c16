"""Host-side mirror of the reference loss-step interface over the C ABI (include/fastclip_b200.h).

The reference drives the step through C++ namespace calls from Trainer::run
(trainer.cpp:427-589); this module exposes the same step as one object per rank:

    cfg  = config_defaults("fastclip_v3", n_train, dim=512, local_batch=5120)
    step = LossStep(cfg)                        # UTable / IndividualTemp / Replica tau in HBM
    de1, de2 = step.step(e1, e2, ids, gamma, eps)   # bf16 [Bl, d] CUDA tensors, int32 ids
    s = step.scalars()                          # loss, G_tau, tau, clamps, latch

There is no CPU fallback: every call goes to the sm_100a kernels in lib/libfastclip_b200.so,
and a missing or unloadable library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

VARIANTS = {
    "openclip_mbcl": 0, "sogclr": 1, "isogclr": 2, "fastclip_v0": 3, "fastclip_v1": 4,
    "fastclip_v2": 5, "fastclip_v3": 6,
}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}

ERRORS = {
    1: "ConfigError", 2: "ShapeError", 3: "DegenerateBatchError", 4: "DomainError",
    5: "OwnershipViolation", 6: "StalenessError", 7: "CollectiveShapeError",
    8: "CollectiveAborted", 9: "NumericError", 10: "IoError", 11: "CudaError", 12: "NcclError",
    13: "Unsupported",
}


class FastclipError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, 'Error')} ({code}): {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "Error")


class FcConfig(C.Structure):
    _fields_ = [
        ("variant", C.c_int32), ("n_train", C.c_int64), ("dim", C.c_int32),
        ("local_batch", C.c_int32), ("world", C.c_int32), ("rank", C.c_int32),
        ("tau_init", C.c_double), ("tau0", C.c_double), ("rho", C.c_double),
        ("tau_lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
        ("adam_eps", C.c_double), ("lr_decay_enabled", C.c_int32),
        ("lr_decay_threshold", C.c_double), ("lr_decay_factor", C.c_double),
        ("scale_by_tau", C.c_int32), ("device", C.c_int32), ("nccl_id", C.c_uint8 * 128),
        ("reduction", C.c_int32),
    ]


class FcStepIn(C.Structure):
    _fields_ = [("e1", C.c_void_p), ("e2", C.c_void_p), ("ids", C.c_void_p),
                ("gamma", C.c_double), ("eps", C.c_double)]


class FcStepOut(C.Structure):
    _fields_ = [("de1", C.c_void_p), ("de2", C.c_void_p)]


class FcStepScalars(C.Structure):
    _fields_ = [("loss", C.c_double), ("gtau", C.c_double), ("tau", C.c_double),
                ("exp_clamps", C.c_uint64), ("latched", C.c_int32)]


class FcLedgerEntry(C.Structure):
    _fields_ = [("phase", C.c_char * 24), ("primitive", C.c_int32), ("world", C.c_int32),
                ("elements", C.c_uint64), ("bytes", C.c_uint64)]


class FcModelState(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("next_epoch", C.c_int64), ("global_step", C.c_int64),
                ("image_shape", C.c_int32 * 4), ("text_shape", C.c_int32 * 4), ("n_params", C.c_int64),
                ("params", C.POINTER(C.c_double)), ("opt_m", C.POINTER(C.c_double)),
                ("opt_v", C.POINTER(C.c_double)), ("opt_step", C.c_int64)]


_lib = None


def lib():
    """Loads (building if needed) the in-tree sm_100a library; raises if unavailable."""
    global _lib
    if _lib is None:
        # FC_LIB_PATH: load another build of the same ABI (A/B diagnostics only)
        path = os.environ.get("FC_LIB_PATH") or _build.build()
        if not os.path.exists(path):
            raise FastclipError(11, f"CUDA library missing: {path}")
        L = C.CDLL(path)
        D, I32, I64, P = C.c_double, C.c_int32, C.c_int64, C.c_void_p
        L.fc_config_defaults.argtypes = [I32, I64, C.POINTER(FcConfig)]
        L.fc_gamma_at.restype = D
        L.fc_gamma_at.argtypes = [I32, D, D, I64, I64, I64]
        L.fc_epsilon_at.restype = D
        L.fc_epsilon_at.argtypes = [D, D, I64, I64]
        L.fc_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8 * 128)]
        L.fc_create.argtypes = [C.POINTER(FcConfig), C.POINTER(P)]
        L.fc_destroy.argtypes = [P]
        L.fc_loss_step.argtypes = [P, C.POINTER(FcStepIn), C.POINTER(FcStepOut), P]
        L.fc_step_scalars_get.argtypes = [P, C.POINTER(FcStepScalars)]
        DP = C.POINTER(C.c_double)
        LP = C.POINTER(C.c_int64)
        L.fc_local_views.argtypes = [P, DP, DP, DP, DP, DP, DP]
        L.fc_table_download.argtypes = [P, DP, DP, DP, DP, DP, DP, LP, DP, DP, LP]
        L.fc_table_upload.argtypes = [P, DP, DP, DP, DP, DP, DP, LP, DP, DP, LP]
        L.fc_tau_state_get.argtypes = [P, DP, DP, DP, LP, C.POINTER(C.c_int32)]
        L.fc_tau_state_set.argtypes = [P, D, D, D, I64, I32]
        L.fc_kernels_per_step.argtypes = [P]
        L.fc_set_phase_timing.argtypes = [P, I32]
        L.fc_phase_times.argtypes = [P, I32, C.POINTER(C.c_float), I32]
        L.fc_debug_similarity.argtypes = [P, P, I32, I32, I32, P, P]
        L.fc_g_values.argtypes = [P, P, I32, I32, P, P, I32, I32, P, P, P, P, P, P]
        L.fc_embedding_cotangents.argtypes = [P, P, I32, I32, P, P, P, P, I32, I32, P, P, P]
        L.fc_temperature_step.argtypes = [DP, DP, LP, D, D, D, D, D, D, D, DP]
        L.fc_table_update.argtypes = [P, P, I64, P, P, P, I32, D, P, P, P, P]
        L.fc_grad_tau.argtypes = [I32, I32, I64, P, P, P, P, P, P, D, D, D, I64, P, P, P, P]
        L.fc_last_error.restype = C.c_char_p
        try:
            _bind_extended(L, D, I32, I64, P, LP)
        except AttributeError:
            if not os.environ.get("FC_LIB_PATH"):   # an older build loaded for an A/B lacks these
                raise
        _lib = L
    return _lib


def _bind_extended(L, D, I32, I64, P, LP):
    if True:
        L.fc_table_write.argtypes = [P, C.c_char_p]
        L.fc_table_read.argtypes = [P, C.c_char_p]
        L.fc_checkpoint_write.argtypes = [P, C.c_char_p, C.POINTER(FcModelState)]
        L.fc_checkpoint_read.argtypes = [P, C.c_char_p, C.POINTER(FcModelState)]
        L.fc_batch_plan_create.argtypes = [I64, I32, C.c_uint64, C.POINTER(P)]
        L.fc_batch_plan_destroy.argtypes = [P]
        L.fc_batch_plan_iters_per_epoch.argtypes = [P]
        L.fc_batch_plan_iters_per_epoch.restype = I64
        L.fc_batch_plan_permutation.argtypes = [P, I64, C.POINTER(C.c_int32)]
        L.fc_batch_plan_local.argtypes = [P, I64, I64, I32, I32, C.POINTER(C.c_int32)]
        L.fc_plan_last_error.restype = C.c_char_p
        L.fc_tower_forward.argtypes = [I32, I32, I32, I32, I32, P, P, P, P, P, P, P, P, P]
        L.fc_tower_vjp.argtypes = [I32, I32, I32, I32, I32, P, P, P, P, P, P, P, P]
        L.fc_grad_allreduce_mean.argtypes = [P, P, I64, P]
        L.fc_adamw_step.argtypes = [I64, P, P, P, LP, P, D, D, D, D, D, P, P]
        L.fc_lamb_step.argtypes = [I64, P, P, P, LP, P, D, D, D, D, D, I32, LP, LP, I32, P, P]
        L.fc_model_last_error.restype = C.c_char_p
        L.fc_comm_ledger.argtypes = [P, C.POINTER(FcLedgerEntry), I32]
        L.fc_comm_ledger_reset.argtypes = [P]


EXPORTED = [
    "fc_config_defaults", "fc_gamma_at", "fc_epsilon_at", "fc_nccl_unique_id", "fc_create",
    "fc_destroy", "fc_loss_step", "fc_step_scalars_get", "fc_local_views", "fc_table_download",
    "fc_table_upload", "fc_tau_state_get", "fc_tau_state_set", "fc_kernels_per_step",
    "fc_debug_similarity", "fc_last_error", "fc_set_phase_timing", "fc_phase_times", "fc_g_values",
    "fc_embedding_cotangents", "fc_temperature_step", "fc_table_update",
    "fc_grad_tau", "fc_table_write", "fc_table_read", "fc_checkpoint_write", "fc_checkpoint_read",
    "fc_batch_plan_create", "fc_batch_plan_destroy", "fc_batch_plan_iters_per_epoch", "fc_batch_plan_permutation",
    "fc_batch_plan_local", "fc_plan_last_error", "fc_synthetic_embeddings", "fc_synthetic_ids", "fc_synthetic_warm_u",
    "fc_tower_forward", "fc_tower_vjp", "fc_grad_allreduce_mean", "fc_adamw_step", "fc_lamb_step",
    "fc_model_last_error", "fc_comm_ledger", "fc_comm_ledger_reset",
]
PHASES = ["allgather_e", "prep", "pass1_stats", "tables_tau", "pass2_q", "grad_gemm"]


def _check(rc: int):
    if rc != 0:
        raise FastclipError(rc, lib().fc_last_error().decode(errors="replace"))


def config_defaults(variant, n_train: int, **fields) -> FcConfig:
    """resolve_algo_config's defaults for the loss step (trainer.cpp:139-194)."""
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    cfg = FcConfig()
    _check(lib().fc_config_defaults(v, int(n_train), C.byref(cfg)))
    for k, val in fields.items():
        setattr(cfg, k, val)
    return cfg


def gamma_at(t: int, *, cosine: bool = True, constant: float = 0.6, gamma_min: float = 0.2,
             decay_epochs: int = 1, iters_per_epoch: int = 1) -> float:
    """GammaSchedule::at (schedules.cpp:25-31)."""
    return lib().fc_gamma_at(int(cosine), constant, gamma_min, decay_epochs, iters_per_epoch, t)


def epsilon_at(epoch: int, initial: float = 1e-14, late: float = 1e-14, switch_epoch: int = -1) -> float:
    """EpsilonSchedule::at (schedules.cpp:62-65)."""
    return lib().fc_epsilon_at(initial, late, switch_epoch, epoch)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().fc_nccl_unique_id(C.byref(buf)))
    return bytes(buf)


@dataclass
class StepScalars:
    loss: float
    gtau: float
    tau: float
    exp_clamps: int
    latched: int


def _dptr(t) -> int:
    return int(t.data_ptr())


class LossStep:
    """One rank of the FastCLIP loss step (trainer.cpp:427-589) on a B200."""

    def __init__(self, cfg: FcConfig):
        self.cfg = cfg
        self._h = C.c_void_p()
        _check(lib().fc_create(C.byref(cfg), C.byref(self._h)))
        self.variant = VARIANT_NAMES[cfg.variant]
        self.individual = cfg.variant in (2, 5)
        self._out = None

    def close(self):
        if self._h:
            lib().fc_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernels_per_step(self) -> int:
        return lib().fc_kernels_per_step(self._h)

    def step(self, e1, e2, ids, gamma: float, eps: float, de1=None, de2=None, stream=None):
        """Enqueues one step on ``stream`` (default: torch's current stream)."""
        import torch
        bl, d = self.cfg.local_batch, self.cfg.dim
        for name, t in (("e1", e1), ("e2", e2)):
            if t.dtype != torch.bfloat16 or not t.is_cuda or tuple(t.shape) != (bl, d) or not t.is_contiguous():
                raise FastclipError(2, f"{name} must be a contiguous CUDA bf16 tensor of shape ({bl}, {d})")
        if ids.dtype != torch.int32 or not ids.is_cuda or ids.numel() != bl:
            raise FastclipError(2, f"ids must be a CUDA int32 tensor with {bl} entries")
        if de1 is None or de2 is None:
            if self._out is None:
                self._out = (torch.empty(bl, d, device=e1.device, dtype=torch.float32),
                             torch.empty(bl, d, device=e1.device, dtype=torch.float32))
            de1, de2 = self._out
        if stream is None:
            stream = torch.cuda.current_stream(e1.device)
        sin = FcStepIn(_dptr(e1), _dptr(e2), _dptr(ids), float(gamma), float(eps))
        sout = FcStepOut(_dptr(de1), _dptr(de2))
        _check(lib().fc_loss_step(self._h, C.byref(sin), C.byref(sout), C.c_void_p(stream.cuda_stream)))
        return de1, de2

    def enable_phase_timing(self, slots: int = 1):
        _check(lib().fc_set_phase_timing(self._h, slots))

    def disable_phase_timing(self):
        _check(lib().fc_set_phase_timing(self._h, 0))

    def phase_times(self, slot: int = -1) -> dict:
        ms = (C.c_float * len(PHASES))()
        _check(lib().fc_phase_times(self._h, slot, ms, len(PHASES)))
        return dict(zip(PHASES, list(ms)))

    def scalars(self) -> StepScalars:
        s = FcStepScalars()
        _check(lib().fc_step_scalars_get(self._h, C.byref(s)))
        return StepScalars(s.loss, s.gtau, s.tau, int(s.exp_clamps), int(s.latched))

    def local_views(self) -> dict:
        n = self.cfg.local_batch
        arrs = {k: np.zeros(n) for k in ("g1", "g2", "u1", "u2", "t1", "t2")}
        p = [arrs[k].ctypes.data_as(C.POINTER(C.c_double)) for k in ("g1", "g2", "u1", "u2", "t1", "t2")]
        _check(lib().fc_local_views(self._h, *p))
        return arrs

    def tables(self) -> dict:
        n = self.cfg.n_train
        t = {"u1": np.zeros(n), "u2": np.zeros(n)}
        if self.individual:
            t.update(tau1=np.zeros(n), tau2=np.zeros(n), m1=np.zeros(n), v1=np.zeros(n),
                     s1=np.zeros(n, np.int64), m2=np.zeros(n), v2=np.zeros(n), s2=np.zeros(n, np.int64))
        _check(lib().fc_table_download(self._h, *self._tab_ptrs(t)))
        return t

    def load_tables(self, **t):
        n = self.cfg.n_train
        full = {}
        for k in ("u1", "u2", "tau1", "tau2", "m1", "v1", "s1", "m2", "v2", "s2"):
            if k in t and t[k] is not None:
                dt = np.int64 if k in ("s1", "s2") else np.float64
                a = np.ascontiguousarray(t[k], dtype=dt)
                if a.shape != (n,):
                    raise FastclipError(10, f"table {k} must have {n} entries")
                full[k] = a
        _check(lib().fc_table_upload(self._h, *self._tab_ptrs(full)))

    @staticmethod
    def _tab_ptrs(t):
        out = []
        for k in ("u1", "u2", "tau1", "tau2", "m1", "v1", "s1", "m2", "v2", "s2"):
            a = t.get(k)
            typ = C.c_int64 if k in ("s1", "s2") else C.c_double
            out.append(a.ctypes.data_as(C.POINTER(typ)) if a is not None else None)
        return out

    def write_tables(self, path: str):
        """UTable::write (+ IndividualTemp::write) of the device tables (state.cpp:73-76, :133-144)."""
        _check(lib().fc_table_write(self._h, os.fsencode(path)))

    def read_tables(self, path: str):
        """UTable::read (+ IndividualTemp::read) into the device tables (state.cpp:87-95, :146-162)."""
        _check(lib().fc_table_read(self._h, os.fsencode(path)))

    def write_checkpoint(self, path: str, model: dict | None = None):
        """write_checkpoint (checkpoint.cpp:57-82): FCK1 with the caller's model part (dict with
        seed, next_epoch, global_step, image_shape, text_shape, params, opt_m, opt_v, opt_step)."""
        ms, keep = _model_state(model)
        _check(lib().fc_checkpoint_write(self._h, os.fsencode(path), C.byref(ms)))
        del keep

    def read_checkpoint(self, path: str) -> dict:
        """read_checkpoint (checkpoint.cpp:84-114): restores tau, its Adam state, the latch and the
        tables into this context; returns the model part."""
        probe = FcModelState()
        _check(lib().fc_checkpoint_read(self._h, os.fsencode(path), C.byref(probe)))
        n = probe.n_params
        arrs = {k: np.zeros(n) for k in ("params", "opt_m", "opt_v")}
        ms = FcModelState()
        ms.n_params = n
        for k, a in arrs.items():
            setattr(ms, k, a.ctypes.data_as(C.POINTER(C.c_double)))
        _check(lib().fc_checkpoint_read(self._h, os.fsencode(path), C.byref(ms)))
        return dict(seed=ms.seed, next_epoch=ms.next_epoch, global_step=ms.global_step,
                    image_shape=list(ms.image_shape), text_shape=list(ms.text_shape), opt_step=ms.opt_step, **arrs)

    def comm_ledger(self) -> dict:
        """CommLedger of the steps so far: {phase: (primitive, reference wire elements, peer bytes)}."""
        buf = (FcLedgerEntry * 16)()
        n = lib().fc_comm_ledger(self._h, buf, 16)
        if n < 0:
            raise FastclipError(-n, "comm_ledger")
        return {buf[i].phase.decode(): (buf[i].primitive, buf[i].elements, buf[i].bytes) for i in range(n)}

    def grad_allreduce_mean(self, grad, stream=None):
        """all_reduce_mean "grad-reduce" (trainer.cpp:540-546) of a CUDA fp64 gradient, in place."""
        import torch
        stream = stream or torch.cuda.current_stream(grad.device)
        _check(lib().fc_grad_allreduce_mean(self._h, _dptr(grad), grad.numel(), C.c_void_p(stream.cuda_stream)))

    def tau_state(self) -> dict:
        tau, m, v = C.c_double(), C.c_double(), C.c_double()
        st, lat = C.c_int64(), C.c_int32()
        _check(lib().fc_tau_state_get(self._h, C.byref(tau), C.byref(m), C.byref(v), C.byref(st), C.byref(lat)))
        return dict(tau=tau.value, m=m.value, v=v.value, step=st.value, latched=lat.value)

    def set_tau_state(self, tau: float, m: float = 0.0, v: float = 0.0, step: int = 0, latched: int = 0):
        _check(lib().fc_tau_state_set(self._h, tau, m, v, step, latched))


def _model_state(model: dict | None):
    ms = FcModelState()
    keep = []
    if model:
        ms.seed = int(model.get("seed", 0))
        ms.next_epoch = int(model.get("next_epoch", 0))
        ms.global_step = int(model.get("global_step", 0))
        for k in ("image_shape", "text_shape"):
            getattr(ms, k)[:] = [int(x) for x in model.get(k, (0, 0, 0, 0))]
        n = len(model.get("params", ()))
        ms.n_params = n
        for k in ("params", "opt_m", "opt_v"):
            a = np.ascontiguousarray(model.get(k, np.zeros(n)), dtype=np.float64)
            if a.shape != (n,):
                raise FastclipError(2, f"model {k} must have {n} entries")
            keep.append(a)
            setattr(ms, k, a.ctypes.data_as(C.POINTER(C.c_double)))
        ms.opt_step = int(model.get("opt_step", 0))
    return ms, keep


class BatchPlan:
    """The reference's index stream (BatchPlan, trainer.cpp:206-241) over its RNG streams
    (rng.hpp:14-65), host side: per-epoch permutations and contiguous per-worker slices."""

    def __init__(self, n_train: int, global_batch: int, seed: int):
        self._h = C.c_void_p()
        rc = lib().fc_batch_plan_create(int(n_train), int(global_batch), int(seed), C.byref(self._h))
        if rc:
            raise FastclipError(rc, lib().fc_plan_last_error().decode())
        self.n_train, self.global_batch = int(n_train), int(global_batch)

    def __del__(self):
        try:
            if self._h:
                lib().fc_batch_plan_destroy(self._h)
        except Exception:
            pass

    @property
    def iters_per_epoch(self) -> int:
        return int(lib().fc_batch_plan_iters_per_epoch(self._h))

    def permutation(self, epoch: int) -> np.ndarray:
        out = np.empty(self.n_train, np.int32)
        _check(lib().fc_batch_plan_permutation(self._h, int(epoch), out.ctypes.data_as(C.POINTER(C.c_int32))))
        return out

    def local_batch(self, epoch: int, it: int, worker: int = 0, world: int = 1) -> np.ndarray:
        out = np.empty(self.global_batch // max(world, 1), np.int32)
        rc = lib().fc_batch_plan_local(self._h, int(epoch), int(it), int(worker), int(world),
                                       out.ctypes.data_as(C.POINTER(C.c_int32)))
        if rc:
            raise FastclipError(rc, lib().fc_plan_last_error().decode())
        return out


def g_values(e1g, e2g, t1_local, t2_local, local_begin: int, local_count: int, dtau_sums: bool = True):
    """engine::g_values (engine.cpp:151-176) [+ engine::dtau_sums (engine.cpp:182-204)] for the
    local slice [local_begin, local_begin + local_count) of the global batch (e1g / e2g: CUDA bf16
    [B, d]; t1/t2_local: CUDA fp64 [local_count]) through the step's tcgen05 pass-1 kernel.
    Returns {"g1", "g2"[, "dsum1", "dsum2"], "clamps"} (CUDA fp64 tensors, clamps a Python int)."""
    import torch
    B, d = e1g.shape
    for name, x in (("e1g", e1g), ("e2g", e2g)):
        if x.dtype != torch.bfloat16 or not x.is_cuda or not x.is_contiguous() or tuple(x.shape) != (B, d):
            raise FastclipError(2, f"{name} must be a contiguous CUDA bf16 tensor of shape ({B}, {d})")
    t1 = t1_local.to(device=e1g.device, dtype=torch.float64).contiguous()
    t2 = t2_local.to(device=e1g.device, dtype=torch.float64).contiguous()
    if t1.numel() != local_count or t2.numel() != local_count:
        raise FastclipError(2, f"t1/t2_local must have {local_count} entries")
    out = {k: torch.empty(local_count, device=e1g.device, dtype=torch.float64)
           for k in (("g1", "g2", "dsum1", "dsum2") if dtau_sums else ("g1", "g2"))}
    ncl = torch.zeros(1, device=e1g.device, dtype=torch.int64)
    stream = torch.cuda.current_stream(e1g.device)
    _check(lib().fc_g_values(_dptr(e1g), _dptr(e2g), B, d, _dptr(t1), _dptr(t2), int(local_begin), int(local_count),
                             _dptr(out["g1"]), _dptr(out["g2"]), _dptr(out["dsum1"]) if dtau_sums else None,
                             _dptr(out["dsum2"]) if dtau_sums else None, _dptr(ncl), C.c_void_p(stream.cuda_stream)))
    out["clamps"] = int(ncl.item())
    return out


def embedding_cotangents(e1g, e2g, w1, w2, t1, t2, local_begin: int, local_count: int):
    """engine::embedding_cotangents (engine.cpp:77-121): dE1, dE2 (CUDA fp32 [local_count, d]) of
    the local slice from the PairWeights w1, w2, t1, t2 over G (fp64 [B]), e1g / e2g CUDA bf16
    [B, d], through the step's pass-1 / pass-2 / gradient-GEMM kernels."""
    import torch
    B, d = e1g.shape
    for name, x in (("e1g", e1g), ("e2g", e2g)):
        if x.dtype != torch.bfloat16 or not x.is_cuda or not x.is_contiguous() or tuple(x.shape) != (B, d):
            raise FastclipError(2, f"{name} must be a contiguous CUDA bf16 tensor of shape ({B}, {d})")
    ws = [x.to(device=e1g.device, dtype=torch.float64).contiguous() for x in (w1, w2, t1, t2)]
    if any(x.numel() != B for x in ws):
        raise FastclipError(2, f"w1, w2, t1, t2 must have {B} entries")
    de1 = torch.empty(local_count, d, device=e1g.device, dtype=torch.float32)
    de2 = torch.empty(local_count, d, device=e1g.device, dtype=torch.float32)
    stream = torch.cuda.current_stream(e1g.device)
    _check(lib().fc_embedding_cotangents(_dptr(e1g), _dptr(e2g), B, d, *[_dptr(x) for x in ws], int(local_begin),
                                         int(local_count), _dptr(de1), _dptr(de2), C.c_void_p(stream.cuda_stream)))
    return de1, de2


def temperature_step(state: dict, tau: float, grad: float, lr: float, beta1=0.9, beta2=0.999, eps=1e-8,
                     tau0=0.005) -> float:
    """opt::temperature_step (optimizers.cpp:77-83) on state {"m", "v", "step"} (updated in place)."""
    m, v, st, out = C.c_double(state["m"]), C.c_double(state["v"]), C.c_int64(state["step"]), C.c_double(0.0)
    _check(lib().fc_temperature_step(C.byref(m), C.byref(v), C.byref(st), tau, grad, lr, beta1, beta2, eps, tau0,
                                     C.byref(out)))
    state.update(m=m.value, v=v.value, step=st.value)
    return out.value


def table_update(u1, u2, ids, g1, g2, gamma: float):
    """UTable::update + snapshot (state.cpp:45-71) on CUDA fp64 tables u1/u2 (in place); returns
    (u1 snapshot, u2 snapshot, status) with status the device-detected error code (0 = ok)."""
    import torch
    n = u1.numel()
    cnt = ids.numel()
    o1 = torch.empty(cnt, device=u1.device, dtype=torch.float64)
    o2 = torch.empty(cnt, device=u1.device, dtype=torch.float64)
    status = torch.zeros(1, device=u1.device, dtype=torch.int32)
    stream = torch.cuda.current_stream(u1.device)
    _check(lib().fc_table_update(_dptr(u1), _dptr(u2), n, _dptr(ids), _dptr(g1), _dptr(g2), cnt, gamma, _dptr(o1),
                                 _dptr(o2), _dptr(status), C.c_void_p(stream.cuda_stream)))
    return o1, o2, int(status.item())


def grad_tau(variant, u1, u2, dsum1, dsum2, batch: int, eps: float, rho: float = 0.0, tau: float = 0.0,
             t1=None, t2=None, n_train: int = 0):
    """engine::grad_tau_* (engine.cpp:208-266) from a worker's u snapshot and dtau sums (CUDA fp64):
    a Python float G_tau,k for v0 / v3 / MBCL, or (gt1, gt2) CUDA tensors for v2 / iSogCLR."""
    import torch
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    n = u1.numel()
    indiv = v in (VARIANTS["isogclr"], VARIANTS["fastclip_v2"])
    g = torch.zeros(1, device=u1.device, dtype=torch.float64)
    gt1 = torch.empty(n, device=u1.device, dtype=torch.float64) if indiv else None
    gt2 = torch.empty(n, device=u1.device, dtype=torch.float64) if indiv else None
    stream = torch.cuda.current_stream(u1.device)
    ptr = lambda x: _dptr(x) if x is not None else None
    _check(lib().fc_grad_tau(v, n, int(batch), _dptr(u1), _dptr(u2), _dptr(dsum1), _dptr(dsum2), ptr(t1), ptr(t2), eps,
                             rho, tau, int(n_train), _dptr(g), ptr(gt1), ptr(gt2), C.c_void_p(stream.cuda_stream)))
    return (gt1, gt2) if indiv else float(g.item())


def debug_similarity(a, b):
    """S = a b^T through the pass-1 tcgen05 tile kernel (fp32), for kernel unit tests."""
    import torch
    rows, d = a.shape
    cols = b.shape[0]
    out = torch.empty(rows, cols, device=a.device, dtype=torch.float32)
    stream = torch.cuda.current_stream(a.device)
    _check(lib().fc_debug_similarity(_dptr(a), _dptr(b), rows, cols, d, _dptr(out), C.c_void_p(stream.cuda_stream)))
    return out


# ---- the model-side step after the loss step ----

def _model_check(rc: int):
    if rc != 0:
        raise FastclipError(rc, lib().fc_model_last_error().decode(errors="replace"))


def tower_param_count(kind: int, d_in: int, d_hidden: int, d_out: int) -> int:
    """TowerShape::param_count (encoder.cpp:20-23)."""
    return d_out * d_in + d_out if kind == 0 else d_hidden * d_in + d_hidden + d_out * d_hidden + d_out


def tower_forward(kind: int, theta, x, d_hidden: int, d_out: int):
    """TwoTowerModel::forward (encoder.cpp:98-134) of one tower on CUDA fp64 tensors: returns the
    tape {x, h, z, e, znorm, e_bf16} (e_bf16: the loss step's input)."""
    import torch
    rows, d_in = x.shape
    dev = x.device
    tape = dict(x=x, h=torch.empty(rows, d_hidden, device=dev, dtype=torch.float64) if kind == 1 else None,
                z=torch.empty(rows, d_out, device=dev, dtype=torch.float64),
                e=torch.empty(rows, d_out, device=dev, dtype=torch.float64),
                znorm=torch.empty(rows, device=dev, dtype=torch.float64),
                e_bf16=torch.empty(rows, d_out, device=dev, dtype=torch.bfloat16))
    status = torch.zeros(1, device=dev, dtype=torch.int32)
    st = torch.cuda.current_stream(dev)
    ptr = lambda t: _dptr(t) if t is not None else None
    _model_check(lib().fc_tower_forward(kind, rows, d_in, d_hidden, d_out, _dptr(theta), _dptr(x), ptr(tape["h"]),
                                        _dptr(tape["z"]), _dptr(tape["e"]), _dptr(tape["znorm"]), _dptr(tape["e_bf16"]),
                                        _dptr(status), C.c_void_p(st.cuda_stream)))
    if int(status.item()):
        raise FastclipError(int(status.item()), "forward: pre-normalization embedding is numerically zero")
    return tape


def tower_vjp(kind: int, theta, tape: dict, cot, grad):
    """TwoTowerModel::vjp (encoder.cpp:136-177): accumulates the tower gradient of the fp32
    cotangent `cot` (the loss step's dE) into `grad` (CUDA fp64, the tower's slice)."""
    import torch
    rows, d_out = tape["e"].shape
    d_in = tape["x"].shape[1]
    d_hidden = tape["h"].shape[1] if tape["h"] is not None else 0
    st = torch.cuda.current_stream(cot.device)
    ptr = lambda t: _dptr(t) if t is not None else None
    _model_check(lib().fc_tower_vjp(kind, rows, d_in, d_hidden, d_out, _dptr(theta), _dptr(tape["x"]), ptr(tape["h"]),
                                    _dptr(tape["e"]), _dptr(tape["znorm"]), _dptr(cot.contiguous()), _dptr(grad),
                                    C.c_void_p(st.cuda_stream)))


def adamw_step(theta, m, v, state: dict, grad, lr: float, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0) -> int:
    """opt::adamw_step (optimizers.cpp:33-41) on CUDA fp64 tensors; state {"step"} updated.
    Returns the device status (0, or FC_ERR_NUMERIC for a non-finite gradient)."""
    import torch
    status = torch.zeros(1, device=theta.device, dtype=torch.int32)
    stp = C.c_int64(state["step"])
    st = torch.cuda.current_stream(theta.device)
    _model_check(lib().fc_adamw_step(theta.numel(), _dptr(theta), _dptr(m), _dptr(v), C.byref(stp), _dptr(grad), lr,
                                     beta1, beta2, eps, weight_decay, _dptr(status), C.c_void_p(st.cuda_stream)))
    state["step"] = stp.value
    return int(status.item())


def lamb_step(theta, m, v, state: dict, grad, lr: float, segments, beta1=0.9, beta2=0.999, eps=1e-8,
              weight_decay=0.0, force_alpha_one=False) -> int:
    """opt::lamb_step (optimizers.cpp:43-63) with layer `segments` [(offset, size), ...]."""
    import torch
    status = torch.zeros(1, device=theta.device, dtype=torch.int32)
    off = (C.c_int64 * len(segments))(*[int(o) for o, _ in segments])
    ln = (C.c_int64 * len(segments))(*[int(n) for _, n in segments])
    stp = C.c_int64(state["step"])
    st = torch.cuda.current_stream(theta.device)
    _model_check(lib().fc_lamb_step(theta.numel(), _dptr(theta), _dptr(m), _dptr(v), C.byref(stp), _dptr(grad), lr,
                                    beta1, beta2, eps, weight_decay, len(segments), off, ln, int(force_alpha_one),
                                    _dptr(status), C.c_void_p(st.cuda_stream)))
    state["step"] = stp.value
    return int(status.item())
