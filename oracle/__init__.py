"""TEST INFRASTRUCTURE: ctypes bindings to the CPU checkers.

* ``ref()``    -- oracle/_ref/libecco_ref.so, the unmodified reference core
                  library (built from /root/reference by oracle/Makefile).
* ``oracle()`` -- oracle/libecco_oracle.so, the plain-C restatement
                  (ecco_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  The product (paper_2512_11727_b200) never
does: it fails loudly when its CUDA library is missing instead of falling
back to anything in here.
"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libecco_ref.so")
ORACLE_SO = os.path.join(HERE, "libecco_oracle.so")
REFERENCE_ROOT = "/root/reference/proj"

_ref = None
_orc = None

dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def build(ref=True):
    """Builds libecco_oracle.so and, where /root/reference exists, libecco_ref.so."""
    targets = ["oracle"]
    if ref and os.path.isdir(REFERENCE_ROOT):
        targets.append("ref")
        if os.path.exists(os.path.join(HERE, "..", "paper_2512_11727_b200", "libecco_b200.so")):
            targets += ["dropin", "unit"]
    subprocess.run(["make", "-s", "-C", HERE, "-j8"] + targets, check=True)


def have_ref():
    return os.path.exists(REF_SO)


class OrcParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("learning_rate_k", "similarity_lambda", "acc_floor", "acc_ceil",
                 "cluster_similarity_threshold")]


class OrcLcfg(C.Structure):
    _fields_ = [("F", C.c_int), ("H", C.c_int), ("C", C.c_int), ("D", C.c_int),
                ("B", C.c_int), ("R", C.c_int), ("S", C.c_int), ("lr", C.c_float),
                ("noise", C.c_float), ("steps_per_gpu_s", C.c_double), ("seed", C.c_uint64)]


def default_params(**kw):
    p = dict(learning_rate_k=0.05, similarity_lambda=0.5, acc_floor=0.1, acc_ceil=0.6,
             cluster_similarity_threshold=0.9)
    p.update(kw)
    return p


def params_array(p):
    return np.array([p["learning_rate_k"], p["similarity_lambda"], p["acc_floor"],
                     p["acc_ceil"], p["cluster_similarity_threshold"]], dtype=np.float64)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO + " (run oracle.build() where /root/reference exists)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_similarity.restype = C.c_double
        L.ref_similarity.argtypes = [dp, dp, C.c_int, C.c_double]
        L.ref_find_cluster.restype = C.c_int
        L.ref_find_cluster.argtypes = [C.c_int, dp, dp, C.c_int, dp, dp]
        L.ref_eval.restype = C.c_double
        L.ref_eval.argtypes = [C.c_int, dp, dp, C.c_int, dp, C.c_int, dp, dp]
        L.ref_eval_matrix.restype = C.c_double
        L.ref_eval_matrix.argtypes = [C.c_int, dp, C.c_int, ip, dp, dp, ip, dp, C.c_int,
                                      C.c_int, dp, dp]
        L.ref_train_step.restype = C.c_int
        L.ref_train_step.argtypes = [C.POINTER(C.c_int), dp, dp, C.POINTER(C.c_int), dp,
                                     C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_int, dp, dp, dp, dp]
        L.ref_seed_model.argtypes = [dp, C.c_int, C.c_double, dp, dp, dp]
        L.ref_profile_table.restype = C.c_int
        L.ref_profile_table.argtypes = [dp, C.c_int, C.c_double, C.c_int, C.c_int, dp, C.c_int,
                                        dp, dp, C.c_double, C.c_double, C.c_double, C.c_double,
                                        dp, dp, dp, dp, u8p]
        L.ref_simulate_window.restype = C.c_int
        L.ref_simulate_window.argtypes = [C.c_int, dp, dp, dp, C.c_double, C.c_double,
                                          C.c_double, dp]
        L.ref_allocate_trajectories.restype = C.c_int
        L.ref_allocate_trajectories.argtypes = [C.c_int, ip, ip, dp, C.c_int, C.c_double,
                                                C.c_double, C.c_int, C.c_double, C.c_int,
                                                C.c_int, C.c_int, ip, dp, dp, dp]
        L.ref_run_scenario.restype = C.c_int
        L.ref_run_scenario.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_size_t,
                                       C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t,
                                       C.POINTER(C.c_size_t)]
        L.ref_time_windows.restype = C.c_int
        L.ref_time_windows.argtypes = [C.c_char_p, C.c_int, dp, C.POINTER(C.c_int)]
        L.ref_time_windows_trace.restype = C.c_int
        L.ref_time_windows_trace.argtypes = [C.c_char_p, C.c_int, dp, C.POINTER(C.c_int),
                                             C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        _ref = L
    return _ref


def oracle():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(ORACLE_SO + " (run oracle.build())")
        L = C.CDLL(ORACLE_SO)
        P = C.POINTER(OrcParams)
        LP = C.POINTER(OrcLcfg)
        L.orc_similarity.restype = C.c_double
        L.orc_similarity.argtypes = [dp, dp, C.c_int, C.c_double]
        L.orc_find_cluster.restype = C.c_int
        L.orc_find_cluster.argtypes = [C.c_int, dp, C.c_int, dp, P]
        L.orc_eval.restype = C.c_double
        L.orc_eval.argtypes = [C.c_int, dp, dp, C.c_int, dp, C.c_int, dp, P]
        L.orc_train_step.restype = C.c_int
        L.orc_train_step.argtypes = [C.POINTER(C.c_int), dp, dp, C.POINTER(C.c_int), dp,
                                     C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_int, dp, dp, dp, P]
        L.orc_seed_model.argtypes = [dp, C.c_int, C.c_double, P, dp, dp]
        L.orc_eval_matrix.argtypes = [C.c_int, dp, C.c_int, ip, dp, dp, ip, dp, C.c_int,
                                      C.c_int, P, dp]
        L.orc_profile_table.restype = C.c_int
        L.orc_profile_table.argtypes = [dp, C.c_int, C.c_double, C.c_int, C.c_int, dp, C.c_int,
                                        dp, dp, C.c_double, C.c_double, C.c_double, C.c_double,
                                        P, dp, dp, dp, u8p]
        L.orc_param_trajectories.restype = C.c_int
        L.orc_param_trajectories.argtypes = [C.c_int, ip, dp, dp, ip, dp, C.c_int, C.c_int, dp,
                                             dp, dp, ip, ip, dp, ip, ip, C.c_double, C.c_int, P,
                                             dp]
        L.orc_philox.argtypes = [u32p, u32p, u32p]
        L.orc_expf.restype = C.c_float
        L.orc_expf.argtypes = [C.c_float]
        L.orc_prototypes.argtypes = [LP, fp, fp]
        L.orc_gen_frames.argtypes = [LP, fp, fp, C.c_int, C.c_int, C.c_int, C.c_int, dp, u16p,
                                     ip]
        L.orc_sample.argtypes = [LP, C.c_int, C.c_int, ip, dp, C.c_int, C.c_int, C.c_int, ip, ip]
        L.orc_init_weights.argtypes = [LP, fp, fp, fp, fp]
        L.orc_sgd_step.restype = C.c_float
        L.orc_sgd_step.argtypes = [LP, u16p, ip, fp, fp, fp, fp]
        L.orc_count_correct.restype = C.c_int
        L.orc_count_correct.argtypes = [LP, u16p, ip, C.c_int, fp, fp, fp, fp]
        L.orc_learned_steps.restype = C.c_int
        L.orc_learned_steps.argtypes = [LP, C.c_double, C.c_double, C.c_double, C.c_double,
                                        C.c_int, dp]
        _orc = L
    return _orc


def orc_params(p):
    return C.byref(OrcParams(**p))
