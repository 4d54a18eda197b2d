"""B200-native group-retraining path of ECCO (arXiv 2512.11727).

Python host mirror of the C-ABI in include/ecco_b200.h.  The compute lives in
``libecco_b200.so`` (hand-written sm_100a CUDA kernels + the C++ window
driver); this module only binds it.  There is no CPU fallback: importing the
package without the built library, or calling into it without a GPU, raises.

Names follow the reference interfaces the entry points replace
(proj/core/include/ecco/*.hpp): ``Context.eval_jobs`` is a batch of
``TrainingBackend::evaluate``, ``Context.eval_matrix`` a batch of
``ModelEvalFn``, ``Context.train_trajectories`` the allocator's
evaluate/train/evaluate probes, ``Context.profile_tables`` the ``ProbeFn`` grid
of ``build_profile_table``, and ``Simulation`` the window loop of
``ecco::Simulation``.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# (ECCO_LIB_PATH: an instrumented build for the tools/ probes; never set by tests or bench)
LIB_PATH = os.environ.get("ECCO_LIB_PATH") or os.path.join(HERE, "libecco_b200.so")

OK, INVALID_ARGUMENT, LOGIC, INFEASIBLE, SCHEMA, CUDA, RUNTIME = range(7)
PARAMETRIC, LEARNED = 0, 1
FFMA_EXACT, TC_BF16 = 0, 1
TC_TF32 = TC_BF16  # round-1 name of the tensor-core mode (ecco_math in include/ecco_b200.h)
# ecco_kstat (include/ecco_b200.h)
(KSTAT_TRAIN_STEP, KSTAT_TRAIN_DW1, KSTAT_TRAIN_HEAD, KSTAT_EVAL_MATRIX, KSTAT_EVAL_PAIRS,
 KSTAT_P_EVAL, KSTAT_P_TRAJ, KSTAT_P_PROFILE, KSTAT_FRAMES) = range(9)


class EccoError(RuntimeError):
    """Base of the errors raised for a non-OK ecco_status."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(EccoError, ValueError):
    """std::invalid_argument in the reference."""


class LogicError(EccoError):
    """std::logic_error in the reference."""


class InfeasibleScheduleError(EccoError):
    """ecco::InfeasibleScheduleError in the reference."""


class SchemaError(EccoError, ValueError):
    """ecco::SchemaError in the reference."""


class CudaError(EccoError):
    pass


_ERRORS = {INVALID_ARGUMENT: InvalidArgument, LOGIC: LogicError, INFEASIBLE: InfeasibleScheduleError,
           SCHEMA: SchemaError, CUDA: CudaError, RUNTIME: EccoError}


class ModelParams(C.Structure):
    _fields_ = [("learning_rate_k", C.c_double), ("similarity_lambda", C.c_double),
                ("acc_floor", C.c_double), ("acc_ceil", C.c_double),
                ("cluster_similarity_threshold", C.c_double)]


class Config(C.Structure):
    _fields_ = [("backend", C.c_int), ("device", C.c_int), ("scene_dims", C.c_int),
                ("max_clusters", C.c_int), ("max_jobs", C.c_int), ("max_cameras", C.c_int),
                ("params", ModelParams), ("math", C.c_int), ("feat_dim", C.c_int),
                ("hidden_dim", C.c_int), ("num_classes", C.c_int), ("minibatch", C.c_int),
                ("ring_frames", C.c_int), ("eval_samples", C.c_int), ("max_depth", C.c_int),
                ("sgd_lr", C.c_float), ("feature_noise", C.c_float),
                ("steps_per_gpu_s", C.c_double), ("seed", C.c_uint64)]


class Batch(C.Structure):
    _fields_ = [("delivered_frame_rate", C.c_double), ("resolution", C.c_double),
                ("quality_factor", C.c_double)]


class SimOptions(C.Structure):
    _fields_ = [("backend", C.c_int), ("math", C.c_int), ("device", C.c_int),
                ("spec_depth", C.c_int), ("feat_dim", C.c_int), ("hidden_dim", C.c_int),
                ("num_classes", C.c_int), ("minibatch", C.c_int), ("ring_frames", C.c_int),
                ("eval_samples", C.c_int), ("sgd_lr", C.c_float),
                ("steps_per_gpu_s", C.c_double), ("seed", C.c_uint64),
                ("host_frames", C.c_int), ("full_matrix", C.c_int)]


_lib = None

# Every symbol include/ecco_b200.h declares (checked by tests/test_abi.py).
# ecco_swap_frame_parts masks
FRAMES_RINGS, FRAMES_EVAL = 1, 2

EXPORTS = [
    "ecco_default_config", "ecco_create", "ecco_destroy", "ecco_last_error",
    "ecco_kernel_launches", "ecco_profile", "ecco_kernel_stat", "ecco_transfer_bytes", "ecco_stream", "ecco_synchronize", "ecco_set_cameras",
    "ecco_update_scenes", "ecco_generate_frames", "ecco_upload_frames", "ecco_upload_frames_dev",
    "ecco_read_frames", "ecco_stage_frames", "ecco_stage_frames_range", "ecco_stage_sampled_frames", "ecco_fetch_sampled_frames",
    "ecco_swap_frames", "ecco_swap_frame_parts", "ecco_reserve_ingest",
    "ecco_put_models", "ecco_get_models", "ecco_seed_models", "ecco_drop_models",
    "ecco_get_weights", "ecco_set_weights", "ecco_eval_jobs", "ecco_eval_matrix",
    "ecco_eval_matrix_dev", "ecco_eval_matrix_dev_async", "ecco_matrix_join", "ecco_eval_pairs", "ecco_rename_models", "ecco_route_propose",
    "ecco_route_matrix_dev", "ecco_route_matrix_ids_dev", "ecco_debug_eval_logits",
    "ecco_train_trajectories", "ecco_commit", "ecco_last_losses", "ecco_sample_indices",
    "ecco_profile_tables", "ecco_sim_default_options", "ecco_sim_create", "ecco_sim_destroy",
    "ecco_sim_last_error", "ecco_sim_step_window", "ecco_sim_last_timings",
    "ecco_sim_last_samples", "ecco_sim_trace_csv", "ecco_sim_summary_json", "ecco_sim_context",
    "ecco_sim_last_timings_ex", "ecco_netsim_mean_rates", "ecco_allocate_trajectories",
]


def netsim_mean_rates(alpha, beta, caps, capacity, rtt_s, duration_s):
    """simulate_window's per-flow mean rates (netsim.cpp:64-94), host code of
    libecco_b200.so: returns (mean rates, steps that needed the sequential
    congestion sum).  Raises InvalidArgument as the reference does."""
    a = np.ascontiguousarray(alpha, np.float64)
    b = np.ascontiguousarray(beta, np.float64)
    c = np.ascontiguousarray(caps, np.float64)
    out = np.zeros(a.size)
    ex = C.c_int()
    st = lib().ecco_netsim_mean_rates(a.size, a, b, c, float(capacity), float(rtt_s),
                                      float(duration_s), out, C.byref(ex))
    if st:
        raise _ERRORS.get(st, EccoError)(st, "netsim: invalid argument")
    return out, ex.value


def allocate_trajectories(job_ids, members, traj, alpha=1.0, beta=1.0, micro_windows=10,
                          micro_s=6.0, gpu_count=1, bonus=True, policy=0):
    """The window driver's allocator decisions (WindowAllocation,
    gpu_allocator.cpp:100-181) on fixed accuracy trajectories: returns
    (jobs, before, after, initial scores)."""
    ids = np.ascontiguousarray(job_ids, np.int32)
    mem = np.ascontiguousarray(members, np.int32)
    t = np.ascontiguousarray(traj, np.float64)
    n, L = t.shape
    job = np.zeros(micro_windows, np.int32)
    b, a, init = np.zeros(micro_windows), np.zeros(micro_windows), np.zeros(n)
    vp = C.c_void_p
    st = lib().ecco_allocate_trajectories(
        n, vp(ids.ctypes.data), vp(mem.ctypes.data), vp(t.ctypes.data), L, C.c_double(alpha),
        C.c_double(beta), micro_windows, C.c_double(micro_s), gpu_count, int(bonus), policy,
        vp(job.ctypes.data), vp(b.ctypes.data), vp(a.ctypes.data), vp(init.ctypes.data))
    if st:
        raise _ERRORS.get(st, EccoError)(st, "allocate_trajectories")
    return job, b, a, init


def lib():
    """Loads libecco_b200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                              "(there is no CPU fallback for the CUDA path)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.ecco_default_config.argtypes = [C.POINTER(Config)]
        L.ecco_create.argtypes = [C.POINTER(Config), C.POINTER(vp)]
        L.ecco_destroy.argtypes = [vp]
        L.ecco_last_error.restype = C.c_char_p
        L.ecco_last_error.argtypes = [vp]
        L.ecco_kernel_launches.restype = C.c_uint64
        L.ecco_kernel_launches.argtypes = [vp]
        L.ecco_stream.restype = vp
        L.ecco_netsim_mean_rates.argtypes = [C.c_int] + [np.ctypeslib.ndpointer(np.float64)] * 3 + [
            C.c_double] * 3 + [np.ctypeslib.ndpointer(np.float64), C.POINTER(C.c_int)]
        L.ecco_stream.argtypes = [vp]
        L.ecco_sim_default_options.argtypes = [C.POINTER(SimOptions)]
        L.ecco_sim_create.argtypes = [C.c_char_p, C.POINTER(SimOptions), C.POINTER(vp),
                                      C.c_char_p, C.c_size_t]
        L.ecco_sim_destroy.argtypes = [vp]
        L.ecco_sim_last_error.restype = C.c_char_p
        L.ecco_sim_last_error.argtypes = [vp]
        L.ecco_sim_step_window.argtypes = [vp, C.POINTER(C.c_int)]
        L.ecco_sim_last_timings.argtypes = [vp, C.POINTER(C.c_double)]
        L.ecco_sim_last_samples.restype = C.c_int64
        L.ecco_sim_last_samples.argtypes = [vp]
        L.ecco_sim_trace_csv.restype = C.c_size_t
        L.ecco_sim_trace_csv.argtypes = [vp, C.c_char_p, C.c_size_t]
        L.ecco_sim_summary_json.restype = C.c_size_t
        L.ecco_sim_summary_json.argtypes = [vp, C.c_char_p, C.c_size_t]
        L.ecco_sim_context.restype = vp
        L.ecco_sim_context.argtypes = [vp]
        for name in EXPORTS:
            f = getattr(L, name)
            if f.restype is C.c_int or name in ("ecco_synchronize",):
                pass
        _lib = L
    return _lib


def _p(a, dtype):
    """Pointer to a contiguous numpy array of `dtype` (None passes NULL)."""
    if a is None:
        return None, None
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr, arr.ctypes.data_as(C.c_void_p)


def default_config(**kw):
    cfg = Config()
    lib().ecco_default_config(C.byref(cfg))
    for k, v in kw.items():
        if k == "params":
            for pk, pv in v.items():
                setattr(cfg.params, pk, pv)
        else:
            setattr(cfg, k, v)
    return cfg


class Context:
    """One ecco_ctx: device state of one GPU (cameras, job models, streams)."""

    def __init__(self, **kw):
        self.cfg = default_config(**kw)
        self._h = C.c_void_p()
        self._check(lib().ecco_create(C.byref(self.cfg), C.byref(self._h)), ctx=False)

    def _check(self, st, ctx=True):
        if st != OK:
            msg = lib().ecco_last_error(self._h).decode() if ctx and self._h else "ecco_create failed"
            raise _ERRORS.get(st, EccoError)(st, msg)

    def close(self):
        if self._h:
            lib().ecco_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def launches(self):
        return lib().ecco_kernel_launches(self._h)

    @property
    def stream(self):
        return lib().ecco_stream(self._h)

    def synchronize(self):
        self._check(lib().ecco_synchronize(self._h))

    # per-kernel CUDA-event profiling (ecco_profile / ecco_kernel_stat)
    def profile(self, enable=True):
        self._check(lib().ecco_profile(self._h, int(bool(enable))))

    def kernel_stat(self, which):
        """(launches, device ms, algorithmic flops, algorithmic bytes) of one
        tracked kernel family (KSTAT_*), accumulated since profiling began."""
        n, ms, fl, by = C.c_uint64(), C.c_double(), C.c_double(), C.c_double()
        self._check(lib().ecco_kernel_stat(self._h, int(which), C.byref(n), C.byref(ms),
                                           C.byref(fl), C.byref(by)))
        return n.value, ms.value, fl.value, by.value

    def transfer_bytes(self):
        h2d, d2h = C.c_uint64(), C.c_uint64()
        self._check(lib().ecco_transfer_bytes(self._h, C.byref(h2d), C.byref(d2h)))
        return h2d.value, d2h.value

    # camera table
    def set_cameras(self, scenes, throughput):
        s, sp = _p(scenes, np.float64)
        t, tpp = _p(throughput, np.float64)
        self._check(lib().ecco_set_cameras(self._h, len(t), sp, tpp))

    def update_scenes(self, cam_idx, scenes):
        c, cp = _p(cam_idx, np.int32)
        s, sp = _p(scenes, np.float64)
        self._check(lib().ecco_update_scenes(self._h, len(c), cp, sp))

    def generate_frames(self, window):
        self._check(lib().ecco_generate_frames(self._h, int(window)))

    def upload_frames(self, frames, labels, eval_frames, eval_labels):
        f, fp = _p(frames, np.uint16)
        l, lp = _p(labels, np.int32)
        e, ep = _p(eval_frames, np.uint16)
        el, elp = _p(eval_labels, np.int32)
        n = len(l) // self.cfg.ring_frames
        self._check(lib().ecco_upload_frames(self._h, n, fp, lp, ep, elp))

    def read_frames(self, n_cams):
        g = self.cfg
        fr = np.zeros((n_cams, g.ring_frames, g.feat_dim), np.uint16)
        lb = np.zeros((n_cams, g.ring_frames), np.int32)
        ev = np.zeros((n_cams, g.eval_samples, g.feat_dim), np.uint16)
        el = np.zeros((n_cams, g.eval_samples), np.int32)
        self._check(lib().ecco_read_frames(self._h, int(n_cams), *[a.ctypes.data_as(C.c_void_p)
                                                                   for a in (fr, lb, ev, el)]))
        return fr, lb, ev, el

    def upload_frames_host_ptr(self, n_cams, frames_ptr, labels_ptr, eval_ptr, eval_labels_ptr):
        """ecco_upload_frames from caller-owned (e.g. pinned) host buffers."""
        self._check(lib().ecco_upload_frames(self._h, int(n_cams), C.c_void_p(frames_ptr),
                                             C.c_void_p(labels_ptr), C.c_void_p(eval_ptr),
                                             C.c_void_p(eval_labels_ptr)))

    def stage_frames_host_ptr(self, n_cams, frames_ptr, labels_ptr, eval_ptr, eval_labels_ptr):
        """ecco_stage_frames: asynchronous upload into the back buffer."""
        self._check(lib().ecco_stage_frames(self._h, int(n_cams), C.c_void_p(frames_ptr),
                                            C.c_void_p(labels_ptr), C.c_void_p(eval_ptr),
                                            C.c_void_p(eval_labels_ptr)))

    def stage_frames_range_host_ptr(self, ring_first, ring_n, frames_ptr, labels_ptr, eval_n,
                                    eval_ptr, eval_labels_ptr):
        """ecco_stage_frames_range: the rings of cameras [ring_first, ring_first
        + ring_n) (pointers at camera ring_first) and the eval sets of cameras
        [0, eval_n), asynchronously into the back buffer."""
        self._check(lib().ecco_stage_frames_range(
            self._h, int(ring_first), int(ring_n), C.c_void_p(frames_ptr), C.c_void_p(labels_ptr),
            int(eval_n), C.c_void_p(eval_ptr), C.c_void_p(eval_labels_ptr)))

    def stage_sampled_host_ptr(self, p, gpu_seconds, depth, window, frames_ptr, labels_ptr,
                               eval_n, eval_ptr, eval_labels_ptr, micro_base=None):
        """ecco_stage_sampled_frames for the prepare_trajectories() batch `p`:
        the ring rows that train_prepared(p, gpu_seconds, depth, window,
        micro_base) will draw are read zero-copy from the PINNED full frame
        table at frames_ptr ([n_cams][R][F] bf16 bits) into the back buffer,
        with every label and the eval sets of cameras [0, eval_n)."""
        mb = p["mb0"] if micro_base is None else np.ascontiguousarray(micro_base, np.int32)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        self._check(lib().ecco_stage_sampled_frames(
            self._h, p["n"], vp(p["ids"]), p["bt"], vp(p["so"]), vp(p["sc"]), vp(p["sf"]), vp(mb),
            C.c_int(window), C.c_double(gpu_seconds), C.c_int(depth), C.c_void_p(frames_ptr),
            C.c_void_p(labels_ptr), int(eval_n), C.c_void_p(eval_ptr), C.c_void_p(eval_labels_ptr)))

    def fetch_sampled_host_ptr(self, p, gpu_seconds, depth, window, frames_ptr, micro_base=None):
        """ecco_fetch_sampled_frames for the prepare_trajectories() batch `p`:
        tops the CURRENT (sampled) rings up with the rows train_prepared(p,
        ...) will draw, from the pinned frame table at frames_ptr."""
        mb = p["mb0"] if micro_base is None else np.ascontiguousarray(micro_base, np.int32)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        self._check(lib().ecco_fetch_sampled_frames(
            self._h, p["n"], vp(p["ids"]), p["bt"], vp(p["so"]), vp(p["sc"]), vp(p["sf"]), vp(mb),
            C.c_int(window), C.c_double(gpu_seconds), C.c_int(depth), C.c_void_p(frames_ptr)))

    def swap_frames(self):
        self._check(lib().ecco_swap_frames(self._h))

    def reserve_ingest(self):
        """ecco_reserve_ingest: allocate the staged ingest's buffers now."""
        self._check(lib().ecco_reserve_ingest(self._h))

    def swap_frame_parts(self, parts):
        """ecco_swap_frame_parts: FRAMES_RINGS (rings + labels) and/or
        FRAMES_EVAL (eval sets + labels) of the staged ingest become current."""
        self._check(lib().ecco_swap_frame_parts(self._h, int(parts)))

    def upload_frames_dev(self, n_cams, frames_ptr, labels_ptr, eval_ptr, eval_labels_ptr):
        self._check(lib().ecco_upload_frames_dev(self._h, int(n_cams), C.c_void_p(frames_ptr),
                                                 C.c_void_p(labels_ptr), C.c_void_p(eval_ptr),
                                                 C.c_void_p(eval_labels_ptr)))

    # models
    def put_models(self, job_ids, n_clusters, clusters, prof, centroid, centroid_len):
        j, jp = _p(job_ids, np.int32)
        k, kp = _p(n_clusters, np.int32)
        c, cp = _p(clusters, np.float64)
        pr, pp = _p(prof, np.float64)
        ce, cep = _p(centroid, np.float64)
        cl, clp = _p(centroid_len, np.int32)
        self._check(lib().ecco_put_models(self._h, len(j), jp, kp, cp, pp, cep, clp))

    def get_models(self, job_ids):
        j, jp = _p(job_ids, np.int32)
        n, K, D = len(j), self.cfg.max_clusters, self.cfg.scene_dims
        k = np.zeros(n, np.int32)
        c = np.zeros((n, K, D))
        pr = np.zeros((n, K))
        ce = np.zeros((n, D))
        cl = np.zeros(n, np.int32)
        self._check(lib().ecco_get_models(self._h, n, jp, k.ctypes.data_as(C.c_void_p),
                                          c.ctypes.data_as(C.c_void_p), pr.ctypes.data_as(C.c_void_p),
                                          ce.ctypes.data_as(C.c_void_p), cl.ctypes.data_as(C.c_void_p)))
        return k, c, pr, ce, cl

    def seed_models(self, job_ids, scenes=None, device_acc=None):
        j, jp = _p(job_ids, np.int32)
        s, sp = _p(scenes, np.float64)
        a, ap = _p(device_acc, np.float64)
        self._check(lib().ecco_seed_models(self._h, len(j), jp, sp, ap))

    def drop_models(self, job_ids):
        j, jp = _p(job_ids, np.int32)
        self._check(lib().ecco_drop_models(self._h, len(j), jp))

    def rename_models(self, old_ids, new_ids):
        o, op = _p(old_ids, np.int32)
        n, np_ = _p(new_ids, np.int32)
        self._check(lib().ecco_rename_models(self._h, len(o), op, np_))

    def _wshapes(self):
        F, H, Cc = self.cfg.feat_dim, self.cfg.hidden_dim, self.cfg.num_classes
        return (F, H), (H,), (H, Cc), (Cc,)

    def get_weights(self, job_id):
        arrs = [np.zeros(s, np.float32) for s in self._wshapes()]
        self._check(lib().ecco_get_weights(self._h, int(job_id),
                                           *[a.ctypes.data_as(C.c_void_p) for a in arrs]))
        return arrs

    def set_weights(self, job_id, w1, b1, w2, b2):
        arrs = [np.ascontiguousarray(a, np.float32) for a in (w1, b1, w2, b2)]
        self._check(lib().ecco_set_weights(self._h, int(job_id),
                                           *[a.ctypes.data_as(C.c_void_p) for a in arrs]))

    # evaluation
    def eval_jobs(self, job_ids, members):
        """TrainingBackend::evaluate for many jobs; members: list of camera-index lists."""
        j, jp = _p(job_ids, np.int32)
        off = np.zeros(len(members) + 1, np.int32)
        off[1:] = np.cumsum([len(m) for m in members])
        mc = np.array([c for m in members for c in m] or [0], np.int32)
        out = np.zeros(len(j))
        self._check(lib().ecco_eval_jobs(self._h, len(j), jp, off.ctypes.data_as(C.c_void_p),
                                         mc.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
        return out

    def eval_matrix(self, job_ids, scenes=None, cams=None, mask=None):
        j, jp = _p(job_ids, np.int32)
        s, sp = _p(scenes, np.float64)
        c, cp = _p(cams, np.int32)
        m, mp = _p(mask, np.uint8)
        n = len(c) if c is not None else len(s) // self.cfg.scene_dims if s.ndim == 1 else len(s)
        out = np.zeros((n, len(j)))
        self._check(lib().ecco_eval_matrix(self._h, n, sp, cp, len(j), jp, mp,
                                           out.ctypes.data_as(C.c_void_p)))
        return out

    def eval_matrix_dev(self, job_ids, out_ptr, scenes=None, cams=None, mask=None):
        j, jp = _p(job_ids, np.int32)
        s, sp = _p(scenes, np.float64)
        c, cp = _p(cams, np.int32)
        m, mp = _p(mask, np.uint8)
        n = len(c) if c is not None else len(s)
        self._check(lib().ecco_eval_matrix_dev(self._h, n, sp, cp, len(j), jp, mp,
                                               C.c_void_p(out_ptr)))

    def eval_matrix_dev_async(self, job_ids, out_ptr, cams, reserve_sms=8):
        """ecco_eval_matrix_dev_async: the matrix on the context's matrix stream,
        leaving reserve_sms SMs for the context stream; join with matrix_join()."""
        j, jp = _p(job_ids, np.int32)
        c, cp = _p(cams, np.int32)
        self._check(lib().ecco_eval_matrix_dev_async(self._h, len(c), cp, len(j), jp,
                                                     C.c_void_p(out_ptr), int(reserve_sms)))

    def matrix_join(self):
        self._check(lib().ecco_matrix_join(self._h))

    def eval_pairs(self, job_ids, scenes=None, cams=None):
        j, jp = _p(job_ids, np.int32)
        s, sp = _p(scenes, np.float64)
        c, cp = _p(cams, np.int32)
        out = np.zeros(len(j))
        self._check(lib().ecco_eval_pairs(self._h, len(j), sp, cp, jp, out.ctypes.data_as(C.c_void_p)))
        return out

    def route_propose(self, job_ids, req_acc, scenes=None, cams=None, mask=None):
        j, jp = _p(job_ids, np.int32)
        r, rp = _p(req_acc, np.float64)
        s, sp = _p(scenes, np.float64)
        c, cp = _p(cams, np.int32)
        m, mp = _p(mask, np.uint8)
        n = len(r)
        best = np.zeros(n, np.int32)
        acc = np.zeros(n)
        self._check(lib().ecco_route_propose(self._h, n, sp, cp, rp, len(j), jp, mp,
                                             best.ctypes.data_as(C.c_void_p),
                                             acc.ctypes.data_as(C.c_void_p)))
        return best, acc

    def debug_eval_logits(self, job_ids, cams):
        """Logits (+ b2) of the fused evaluation kernel: [n_cams, S, n_jobs, C]."""
        j, jp = _p(job_ids, np.int32)
        c, cp = _p(cams, np.int32)
        g = self.cfg
        out = np.zeros((len(c), g.eval_samples, len(j), g.num_classes), np.float32)
        self._check(lib().ecco_debug_eval_logits(self._h, len(c), cp, len(j), jp,
                                                 out.ctypes.data_as(C.c_void_p)))
        return out

    def route_matrix_dev(self, n, g_block, matrix_ptr, best_ptr, acc_ptr, req_ptr=None,
                         n_blocks=1):
        """Argmax/threshold epilogue over a device matrix (all pointers device)."""
        self._check(lib().ecco_route_matrix_dev(self._h, int(n), int(g_block), int(n_blocks),
                                                C.c_void_p(matrix_ptr),
                                                C.c_void_p(req_ptr) if req_ptr else None,
                                                C.c_void_p(best_ptr), C.c_void_p(acc_ptr)))

    def route_matrix_ids_dev(self, n, g_block, matrix_ptr, ids_ptr, best_ptr, acc_ptr,
                             req_ptr=None, n_blocks=1):
        """ecco_route_matrix_ids_dev: the same epilogue with a device column ->
        group id map (int32, < 0 = padding); best_ptr receives group ids."""
        self._check(lib().ecco_route_matrix_ids_dev(
            self._h, int(n), int(g_block), int(n_blocks), C.c_void_p(matrix_ptr),
            C.c_void_p(ids_ptr), C.c_void_p(req_ptr) if req_ptr else None, C.c_void_p(best_ptr),
            C.c_void_p(acc_ptr)))

    # training
    def prepare_trajectories(self, job_ids, batches, sources, fracs, members):
        """Flattens the per-job arguments of train_trajectories once (CSR
        source_mix / member lists, ecco_batch array) so a caller that trains
        the same jobs every window does no per-call list building."""
        n = len(job_ids)
        p = {"n": n}
        p["ids"] = np.ascontiguousarray(job_ids, np.int32)
        p["bt"] = (Batch * max(n, 1))(*[Batch(*b) for b in batches])
        so = np.zeros(n + 1, np.int32)
        so[1:] = np.cumsum([len(x) for x in sources])
        p["so"] = so
        p["sc"] = np.array([c for x in sources for c in x] or [0], np.int32)
        p["sf"] = np.array([f for x in fracs for f in x] or [0.0], np.float64)
        mo = np.zeros(n + 1, np.int32)
        mo[1:] = np.cumsum([len(m) for m in members])
        p["mo"] = mo
        p["mc"] = np.array([c for m in members for c in m] or [0], np.int32)
        p["mb0"] = np.zeros(max(n, 1), np.int32)
        return p

    def train_prepared(self, p, gpu_seconds, depth, window=0, micro_base=None, out=None):
        """ecco_train_trajectories on a prepare_trajectories() batch; returns
        acc[n_jobs, depth+1] (written into `out` when given)."""
        n = p["n"]
        if out is None:
            out = np.zeros((n, depth + 1))
        mb = p["mb0"] if micro_base is None else np.ascontiguousarray(micro_base, np.int32)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        self._check(lib().ecco_train_trajectories(
            self._h, n, vp(p["ids"]), p["bt"], vp(p["so"]), vp(p["sc"]), vp(p["sf"]), vp(p["mo"]),
            vp(p["mc"]), vp(mb), C.c_int(window), C.c_double(gpu_seconds), C.c_int(depth),
            vp(out)))
        return out

    def train_trajectories(self, job_ids, batches, sources, fracs, members, gpu_seconds, depth,
                           micro_base=None, window=0):
        """Speculative evaluate/train chains.  batches: list of (fps, res, quality);
        sources/fracs: per-job source_mix (camera indices in map order, fractions);
        members: per-job member camera indices.  Returns acc[n_jobs, depth+1]."""
        p = self.prepare_trajectories(job_ids, batches, sources, fracs, members)
        return self.train_prepared(p, gpu_seconds, depth, window=window, micro_base=micro_base)

    def commit(self, job_ids, granted):
        j, jp = _p(job_ids, np.int32)
        g, gp = _p(granted, np.int32)
        self._check(lib().ecco_commit(self._h, len(j), jp, gp))

    def last_losses(self, job_ids, depth):
        j, jp = _p(job_ids, np.int32)
        out = np.zeros((len(j), depth), np.float32)
        self._check(lib().ecco_last_losses(self._h, len(j), jp, int(depth),
                                           out.ctypes.data_as(C.c_void_p)))
        return out

    def sample_indices(self, job_id, src_cams, src_fracs, window, micro, step):
        c, cp = _p(src_cams, np.int32)
        f, fp = _p(src_fracs, np.float64)
        B = self.cfg.minibatch
        oc = np.zeros(B, np.int32)
        of = np.zeros(B, np.int32)
        self._check(lib().ecco_sample_indices(self._h, int(job_id), len(c), cp, fp, int(window),
                                              int(micro), int(step), oc.ctypes.data_as(C.c_void_p),
                                              of.ctypes.data_as(C.c_void_p)))
        return oc, of

    def profile_tables(self, cam_idx, levels, grid_fps, grid_res, window_s, bias=None,
                       tie_eps=1e-9, ref_rate_bps=1e6, bpp_ref=0.1):
        c, cp = _p(cam_idx, np.int32)
        b, bp = _p(bias, np.int32)
        l, lp = _p(levels, np.float64)
        gf, gfp = _p(grid_fps, np.float64)
        gq, gqp = _p(grid_res, np.float64)
        rows = (len(c), len(l))
        ob, of, oq = np.zeros(rows), np.zeros(rows), np.zeros(rows)
        fe = np.zeros(rows, np.uint8)
        self._check(lib().ecco_profile_tables(
            self._h, len(c), cp, bp, len(l), lp, len(gf), gfp, gqp, C.c_double(window_s),
            C.c_double(tie_eps), C.c_double(ref_rate_bps), C.c_double(bpp_ref),
            ob.ctypes.data_as(C.c_void_p), of.ctypes.data_as(C.c_void_p),
            oq.ctypes.data_as(C.c_void_p), fe.ctypes.data_as(C.c_void_p)))
        return ob, of, oq, fe


def default_sim_options(**kw):
    o = SimOptions()
    lib().ecco_sim_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Simulation:
    """ecco::Simulation (orchestrator.hpp:34-73) over the B200 path."""

    def __init__(self, scenario_json, **options):
        if isinstance(scenario_json, dict):
            import json
            scenario_json = json.dumps(scenario_json)
        self.options = default_sim_options(**options)
        self._h = C.c_void_p()
        err = C.create_string_buffer(4096)
        st = lib().ecco_sim_create(scenario_json.encode(), C.byref(self.options), C.byref(self._h),
                                   err, 4096)
        if st != OK:
            raise _ERRORS.get(st, EccoError)(st, err.value.decode())

    def close(self):
        if self._h:
            lib().ecco_sim_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step_window(self):
        ran = C.c_int()
        st = lib().ecco_sim_step_window(self._h, C.byref(ran))
        if st != OK:
            raise _ERRORS.get(st, EccoError)(st, lib().ecco_sim_last_error(self._h).decode())
        return bool(ran.value)

    def run(self):
        while self.step_window():
            pass

    def last_timings(self):
        t = (C.c_double * 11)()
        n = lib().ecco_sim_last_timings_ex(self._h, t, 11)
        return dict(zip(("window_ms", "regroup_ms", "train_ms", "window_end_ms", "replay_ms",
                         "netsim_ms", "profile_ms", "events_ms", "route_ms", "shares_configs_ms",
                         "rows_ms"), list(t)[:n]))

    def last_samples(self):
        return lib().ecco_sim_last_samples(self._h)

    def trace_csv(self):
        n = lib().ecco_sim_trace_csv(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        lib().ecco_sim_trace_csv(self._h, buf, n)
        return buf.raw[:n].decode()

    def summary_json(self):
        n = lib().ecco_sim_summary_json(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        lib().ecco_sim_summary_json(self._h, buf, n)
        return buf.raw[:n].decode()

    @property
    def context_handle(self):
        return lib().ecco_sim_context(self._h)

    @property
    def launches(self):
        return lib().ecco_kernel_launches(self.context_handle)
