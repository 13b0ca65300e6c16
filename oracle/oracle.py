"""ctypes bindings for the CPU checkers -- TEST INFRASTRUCTURE ONLY.

Two interchangeable backends with the same C signature (fastclip_oracle.h):
  * ``oracle``: the plain-C restatement (oracle/fastclip_oracle.c)
  * ``ref``:    the reference's own translation units compiled against the Eigen-subset shim
                (oracle/ref_driver.cpp, built into oracle/_ref/ by oracle/Makefile).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfastclip_ref.so")
REF_FAST_SO = os.path.join(HERE, "_ref", "libfastclip_ref_fast.so")

# Variant ids (trainer.hpp:145-153)
OPENCLIP_MBCL, SOGCLR, ISOGCLR, FASTCLIP_V0, FASTCLIP_V1, FASTCLIP_V2, FASTCLIP_V3 = range(7)
VARIANTS = {
    "openclip_mbcl": OPENCLIP_MBCL, "sogclr": SOGCLR, "isogclr": ISOGCLR,
    "fastclip_v0": FASTCLIP_V0, "fastclip_v1": FASTCLIP_V1, "fastclip_v2": FASTCLIP_V2,
    "fastclip_v3": FASTCLIP_V3,
}


class OcConfig(C.Structure):
    _fields_ = [
        ("variant", C.c_int), ("n_train", C.c_int64), ("tau0", C.c_double), ("rho", C.c_double),
        ("tau_lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
        ("adam_eps", C.c_double), ("lr_decay_enabled", C.c_int),
        ("lr_decay_threshold", C.c_double), ("lr_decay_factor", C.c_double),
        ("scale_by_tau", C.c_int),
    ]


_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int64)


class OcState(C.Structure):
    _fields_ = [
        ("u1", _DP), ("u2", _DP), ("tau1", _DP), ("tau2", _DP),
        ("m1", _DP), ("v1", _DP), ("s1", _IP), ("m2", _DP), ("v2", _DP), ("s2", _IP),
        ("tau", C.c_double), ("tau_m", C.c_double), ("tau_v", C.c_double),
        ("tau_step", C.c_int64), ("latched", C.c_int),
    ]


class OcStepOut(C.Structure):
    _fields_ = [
        ("dE1", _DP), ("dE2", _DP), ("g1", _DP), ("g2", _DP), ("u1", _DP), ("u2", _DP),
        ("t1", _DP), ("t2", _DP), ("gtau1", _DP), ("gtau2", _DP), ("gtau_local", _DP),
        ("gtau", C.c_double), ("tau_new", C.c_double), ("loss", C.c_double),
        ("clamps_g", C.c_uint64),
    ]


def default_config(variant: str, n_train: int, **over) -> dict:
    """Variant defaults as resolved by resolve_algo_config (trainer.cpp:139-194) with the
    RunConfig registry defaults (config.cpp:36-60): tau0=0.005, Adam (0.9, 0.999, 1e-8),
    latch threshold 0.03 and factor 1/3."""
    v = VARIANTS[variant]
    if v in (SOGCLR, FASTCLIP_V1):
        lr = 0.0
    elif v in (ISOGCLR, FASTCLIP_V2):
        lr = 1e-2
    else:
        lr = 2e-4
    if v in (ISOGCLR, FASTCLIP_V2):
        rho = 9.0
    elif v == FASTCLIP_V3:
        rho = 6.5
    else:
        rho = 0.0
    cfg = dict(
        variant=v, n_train=n_train, tau0=0.005, rho=rho, tau_lr=lr, beta1=0.9, beta2=0.999,
        adam_eps=1e-8, lr_decay_enabled=1 if v == FASTCLIP_V3 else 0,
        lr_decay_threshold=0.03, lr_decay_factor=1.0 / 3.0,
        scale_by_tau=0 if v in (FASTCLIP_V0, OPENCLIP_MBCL) else 1,
        tau_init=0.07 if v == FASTCLIP_V3 else 0.03,
    )
    cfg.update(over)
    return cfg


def _ptr(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


@dataclass
class TableState:
    """Dataset-sized run state (u table, v2 tau tables + sparse Adam, global tau)."""
    n: int
    individual: bool
    tau: float
    u1: np.ndarray = field(init=False)
    u2: np.ndarray = field(init=False)

    def __post_init__(self):
        self.u1 = np.zeros(self.n)
        self.u2 = np.zeros(self.n)
        if self.individual:
            self.tau1 = np.full(self.n, self.tau)
            self.tau2 = np.full(self.n, self.tau)
            self.m1 = np.zeros(self.n); self.v1 = np.zeros(self.n); self.s1 = np.zeros(self.n, np.int64)
            self.m2 = np.zeros(self.n); self.v2 = np.zeros(self.n); self.s2 = np.zeros(self.n, np.int64)
        else:
            self.tau1 = self.tau2 = self.m1 = self.v1 = self.s1 = self.m2 = self.v2 = self.s2 = None
        self.tau_m = 0.0
        self.tau_v = 0.0
        self.tau_step = 0
        self.latched = 0

    def copy(self) -> "TableState":
        c = TableState.__new__(TableState)
        c.__dict__.update({k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in self.__dict__.items()})
        return c

    def to_c(self) -> OcState:
        return OcState(_ptr(self.u1), _ptr(self.u2), _ptr(self.tau1), _ptr(self.tau2),
                       _ptr(self.m1), _ptr(self.v1), _ptr(self.s1, C.c_int64),
                       _ptr(self.m2), _ptr(self.v2), _ptr(self.s2, C.c_int64),
                       self.tau, self.tau_m, self.tau_v, self.tau_step, self.latched)

    def from_c(self, st: OcState) -> None:
        self.tau = st.tau; self.tau_m = st.tau_m; self.tau_v = st.tau_v
        self.tau_step = st.tau_step; self.latched = st.latched


def _cfg_c(cfg: dict) -> OcConfig:
    return OcConfig(*[cfg[f] for f, _ in OcConfig._fields_])


_libs: dict = {}


def lib(kind: str = "oracle"):
    path = {"oracle": ORACLE_SO, "ref": REF_SO, "ref_fast": REF_FAST_SO}[kind]
    if kind not in _libs:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        _libs[kind] = L
        D, I = C.c_double, C.c_int
        if kind == "oracle":
            L.oc_step.argtypes = [C.POINTER(OcConfig), C.POINTER(OcState), I, I, I, _DP, _DP,
                                  C.POINTER(C.c_int32), D, D, C.POINTER(OcStepOut)]
            L.oc_safe_exp.restype = D
            L.oc_safe_exp.argtypes = [D]
            L.oc_exp_clamp_count.restype = C.c_uint64
            for f in ("oc_eval_gcl", "oc_eval_mbcl", "oc_eval_rgcl"):
                getattr(L, f).restype = D
            L.oc_gamma_cosine.restype = D
            L.oc_gamma_cosine.argtypes = [C.c_longlong, C.c_longlong, C.c_longlong, D]
            L.oc_epsilon_at.restype = D
            L.oc_epsilon_at.argtypes = [C.c_longlong, D, D, C.c_longlong]
            L.oc_latch_modifier.restype = D
            L.oc_latch_modifier.argtypes = [C.POINTER(C.c_int), D, D, D]
        else:
            L.ref_create.restype = C.c_void_p
            L.ref_create.argtypes = [C.POINTER(OcConfig)]
            L.ref_destroy.argtypes = [C.c_void_p]
            L.ref_set_state.argtypes = [C.c_void_p, C.POINTER(OcState)]
            L.ref_get_state.argtypes = [C.c_void_p, C.POINTER(OcState)]
            L.ref_step_ex.argtypes = [C.c_void_p, I, I, I, _DP, _DP, C.POINTER(C.c_int32), D, D,
                                      C.POINTER(OcStepOut), I, I]
            for f in ("ref_eval_gcl", "ref_eval_mbcl", "ref_eval_rgcl", "ref_safe_exp",
                      "ref_gamma_cosine", "ref_similarity_checksum"):
                getattr(L, f).restype = D
            L.ref_gamma_cosine.argtypes = [C.c_longlong, C.c_longlong, C.c_longlong, D]
            L.ref_safe_exp.argtypes = [D]
            L.ref_exp_clamp_count.restype = C.c_ulonglong
            # ref_next.cpp: the §8(f) rows next to the loss step (state / checkpoint formats, index
            # plan, model optimizers, reduce-scatter pieces, wire model)
            LL, ULL, CP = C.c_longlong, C.c_ulonglong, C.c_char_p
            LP = C.POINTER(C.c_longlong)
            L.ref_tables_write.argtypes = [CP, LL, _DP, _DP, _DP, _DP, D, _DP, _DP, LP, _DP, _DP, LP]
            L.ref_tables_read.argtypes = [CP, LL, I, _DP, _DP, _DP, _DP, _DP, _DP, _DP, LP, _DP, _DP, LP]
            L.ref_checkpoint_rewrite.argtypes = [CP, CP]
            L.ref_checkpoint_fields.argtypes = [CP, C.POINTER(ULL), LP, LP, LP, _DP, _DP, _DP, LP,
                                                C.POINTER(I), C.POINTER(I)]
            L.ref_checkpoint_make.argtypes = [CP, ULL, LL, LL, I, I, LL, _DP, _DP, _DP, LL, D, D, D, LL, I, LL,
                                              _DP, _DP]
            L.ref_batch_plan_local.argtypes = [LL, I, ULL, LL, LL, I, I, C.POINTER(C.c_int)]
            L.ref_stream_seed2.restype = ULL
            L.ref_stream_seed2.argtypes = [ULL, ULL, ULL, I]
            L.ref_rng_normals.argtypes = [ULL, LL, _DP]
            L.ref_rng_below.argtypes = [ULL, LL, ULL, C.POINTER(ULL)]
            L.ref_adamw_step.argtypes = [LL, _DP, _DP, _DP, LP, _DP, D, D, D, D, D]
            L.ref_lamb_step.argtypes = [LL, _DP, _DP, _DP, LP, _DP, D, D, D, D, D, I, LP, LP, I]
            L.ref_rs_partials.argtypes = [I, I, _DP, _DP, _DP, _DP, _DP, _DP, I, I, _DP, _DP]
            L.ref_rs_shard_scale.restype = D
            L.ref_rs_shard_scale.argtypes = [I, I, LL]
            L.ref_wire.restype = ULL
            L.ref_wire.argtypes = [I, I, ULL]
    return _libs[kind]


def new_state(cfg: dict) -> TableState:
    indiv = cfg["variant"] in (ISOGCLR, FASTCLIP_V2)
    return TableState(int(cfg["n_train"]), indiv, float(cfg["tau_init"]))


def _alloc_out(K: int, B: int, d: int):
    arrs = dict(
        dE1=np.zeros((B, d)), dE2=np.zeros((B, d)), g1=np.zeros(B), g2=np.zeros(B),
        u1=np.zeros(B), u2=np.zeros(B), t1=np.zeros(B), t2=np.zeros(B),
        gtau1=np.zeros(B), gtau2=np.zeros(B), gtau_local=np.zeros(K),
    )
    o = OcStepOut(*[_ptr(arrs[k]) for k in ("dE1", "dE2", "g1", "g2", "u1", "u2", "t1", "t2",
                                           "gtau1", "gtau2", "gtau_local")], 0.0, 0.0, 0.0, 0)
    return arrs, o


def step(cfg: dict, state: TableState, K: int, E1: np.ndarray, E2: np.ndarray,
         ids: np.ndarray, gamma: float, eps: float, backend: str = "oracle",
         local_limit: int = 0) -> dict:
    """One loss step (trainer.cpp:427-589) for K workers; updates ``state`` in place."""
    E1 = np.ascontiguousarray(E1, dtype=np.float64)
    E2 = np.ascontiguousarray(E2, dtype=np.float64)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    B, d = E1.shape
    arrs, o = _alloc_out(K, B, d)
    cc = _cfg_c(cfg)
    st = state.to_c()
    if backend == "oracle":
        rc = lib("oracle").oc_step(C.byref(cc), C.byref(st), K, B, d, _ptr(E1), _ptr(E2),
                                   _ptr(ids, C.c_int32), gamma, eps, C.byref(o))
        state.from_c(st)
    else:
        L = lib(backend)
        h = L.ref_create(C.byref(cc))
        try:
            L.ref_set_state(h, C.byref(st))
            rc = L.ref_step_ex(h, K, B, d, _ptr(E1), _ptr(E2), _ptr(ids, C.c_int32), gamma, eps,
                               C.byref(o), local_limit, 0 if local_limit else 1)
            L.ref_get_state(h, C.byref(st))
            state.from_c(st)
        finally:
            L.ref_destroy(h)
    if rc != 0:
        raise RuntimeError(f"{backend} step failed with status {rc}")
    arrs.update(gtau=o.gtau, tau_new=o.tau_new, loss=o.loss, clamps_g=int(o.clamps_g))
    return arrs
