"""Thin ctypes binding of libpas (include/pas.h): the same entry points, argument marshalling only.

Every step of the routing path runs in libpas's CUDA kernels; this module only converts Python /
torch arguments to pointers and sizes.  PyTorch is used for device memory and streams.  If the
library has not been built (``python -m paper_2502_06798_b200.build``) importing this module raises:
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PAS_LIB selects an alternative build of the same C-ABI (kernel A/B experiments only)
LIB_PATH = os.environ.get("PAS_LIB") or os.path.join(_HERE, "lib", "libpas.so")

PAS_OK = 0
STATUS = {0: "PAS_OK", -1: "PAS_ERR_ARG", -2: "PAS_ERR_STATE", -3: "PAS_ERR_FRACTIONS",
          -4: "PAS_ERR_NO_INSTANCE", -5: "PAS_ERR_BANDS", -6: "PAS_ERR_DEGRADATION",
          -7: "PAS_ERR_CAPACITY", -8: "PAS_ERR_CUDA", -9: "PAS_ERR_NCCL", -10: "PAS_ERR_INVALID_ROWS"}
PAS_F32, PAS_BF16 = 0, 1
PAS_GREEDY, PAS_UNIFORM = 0, 1
PAS_MAX_LEVELS, PAS_MAX_INSTANCES, PAS_T_TOTAL, PAS_MAX_TOPK = 16, 64, 50, 16
PAS_MAX_FORECAST_WINDOW = 1 << 22
PAS_NCCL_ID_BYTES = 128
PAS_NEVER_BUSY = -(1 << 62)
FLAG_INVALID, FLAG_COLD, FLAG_NEAR_TOP1, FLAG_NEAR_THRESHOLD = 1, 2, 4, 8


class PasConfig(C.Structure):
    _fields_ = [("d", C.c_int), ("topk", C.c_int), ("max_batch", C.c_int64),
                ("max_rows_per_rank", C.c_int64), ("device", C.c_int), ("rank", C.c_int),
                ("world", C.c_int), ("nccl_id", C.c_void_p), ("seed", C.c_uint64)]


class PasRouteOut(C.Structure):
    _fields_ = [("K", C.c_void_p), ("K_prime", C.c_void_p), ("instance", C.c_void_p),
                ("slot", C.c_void_p), ("topk_id", C.c_void_p), ("topk_score", C.c_void_p),
                ("flags", C.c_void_p), ("bucket_offsets", C.c_void_p), ("bucket_prompts", C.c_void_p)]


class PasStats(C.Structure):
    _fields_ = [("nK", C.c_int), ("W", C.c_int), ("N", C.c_int64),
                ("h", C.c_int64 * PAS_MAX_LEVELS), ("f", C.c_int64 * PAS_MAX_LEVELS),
                ("x", (C.c_int64 * PAS_MAX_LEVELS) * PAS_MAX_LEVELS),
                ("D_Q", C.c_double), ("D_Q_LP", C.c_double), ("plan_solver_iters", C.c_int),
                ("n_redirected", C.c_int64), ("n_upgraded", C.c_int64), ("n_downgraded", C.c_int64),
                ("n_invalid", C.c_int64), ("n_near_top1", C.c_int64), ("n_near_threshold", C.c_int64),
                ("bucket_count", C.c_int64 * PAS_MAX_INSTANCES), ("stage_ms", C.c_float * 8),
                ("forecast", C.c_int), ("fc_replanned", C.c_int), ("fc_plan_n", C.c_int64),
                ("fc_plan_counts", C.c_int64 * PAS_MAX_LEVELS), ("fc_window_n", C.c_int64),
                ("fc_l2_error", C.c_double), ("n_unforecast", C.c_int64),
                ("fc_Hc", C.c_uint64 * (PAS_MAX_LEVELS + 1)), ("fc_Fc", C.c_uint64 * (PAS_MAX_LEVELS + 1)),
                ("dispatcher", C.c_int), ("now_us", C.c_int64),
                ("queue_len", C.c_int64 * PAS_MAX_INSTANCES), ("busy_until_us", C.c_int64 * PAS_MAX_INSTANCES),
                ("fired_prompts", C.c_int64 * PAS_MAX_INSTANCES),
                ("fired_batches", C.c_int64 * PAS_MAX_INSTANCES),
                ("k2_ranges", C.c_int), ("k2_chunk_tiles", C.c_int), ("k2_chunk_steps", C.c_int),
                ("k6_fallback", C.c_int)]


class PasAssignment(C.Structure):
    _fields_ = [("nK", C.c_int), ("W", C.c_int), ("n", C.c_int32 * PAS_MAX_LEVELS),
                ("F", C.c_double * PAS_MAX_LEVELS), ("F_route", C.c_double * PAS_MAX_LEVELS),
                ("H", C.c_double * PAS_MAX_LEVELS), ("served", C.c_double), ("quality", C.c_double),
                ("instance_level", C.c_int32 * PAS_MAX_INSTANCES), ("candidates", C.c_int64),
                ("solve_ms", C.c_float)]


class PasError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"libpas.so is not built ({LIB_PATH}); run `python -m paper_2502_06798_b200.build` "
                      "-- there is no CPU fallback")
lib = C.CDLL(LIB_PATH)

_P = C.c_void_p
_SIG = {
    "pas_version": (C.c_char_p, []),
    "pas_create": (C.c_int, [C.POINTER(_P), C.POINTER(PasConfig)]),
    "pas_destroy": (C.c_int, [_P]),
    "pas_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "pas_cache_load": (C.c_int, [_P, _P, C.c_int, C.c_int64, C.POINTER(C.c_int64), _P]),
    "pas_cache_clear": (C.c_int, [_P]),
    "pas_cache_insert": (C.c_int, [_P, _P, C.c_int, C.c_int64, _P, _P]),
    "pas_cache_insert_vanilla": (C.c_int, [_P, _P, C.c_int, C.c_int64, _P, _P, C.POINTER(C.c_int64), _P]),
    "pas_cache_stamps": (C.c_int, [_P, _P, C.c_int64, _P]),
    "pas_cache_size": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pas_set_bands": (C.c_int, [_P, C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_float)]),
    "pas_set_degradation": (C.c_int, [_P, C.POINTER(C.c_double), C.c_int]),
    "pas_set_fractions": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_int, C.c_int, C.c_int]),
    "pas_set_seed": (C.c_int, [_P, C.c_uint64, C.c_uint64]),
    "pas_set_collectives": (C.c_int, [_P, C.c_int]),
    "pas_set_graph": (C.c_int, [_P, C.c_int]),
    "pas_stage_ring": (C.c_int, [_P, C.c_int]),
    "pas_stage_ring_read": (C.c_int, [_P, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_int)]),
    "pas_set_forecast": (C.c_int, [_P, C.c_int, C.c_int]),
    "pas_set_dispatcher": (C.c_int, [_P, C.POINTER(C.c_int64), C.c_int, C.c_int64]),
    "pas_set_clock": (C.c_int, [_P, C.c_int64]),
    "pas_set_load": (C.c_int, [_P, C.c_double, C.c_int, C.POINTER(C.c_int)]),
    "pas_dispatcher_state": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64)]),
    "pas_solve_assignment": (C.c_int, [_P, C.c_int, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                       C.c_int, C.POINTER(PasAssignment)]),
    "pas_route_batch": (C.c_int, [_P, _P, C.c_int, C.c_int64, C.POINTER(PasRouteOut), _P]),
    "pas_route_batch_host": (C.c_int, [_P, _P, C.c_int, C.c_int64, C.POINTER(PasRouteOut), _P]),
    "pas_route_batch_host_async": (C.c_int, [_P, _P, C.c_int, C.c_int64, C.POINTER(PasRouteOut), _P]),
    "pas_route_host_begin": (C.c_int, [_P, _P]),
    "pas_route_host_end": (C.c_int, [_P, _P]),
    "pas_route_local": (C.c_int, [_P, _P, C.c_int, C.c_int64, _P, _P]),
    "pas_route_from_candidates": (C.c_int, [_P, _P, C.c_int, C.c_int64, C.POINTER(PasRouteOut), _P]),
    "pas_plan_stats": (C.c_int, [_P, C.POINTER(PasStats)]),
    "pas_last_error": (C.c_char_p, [_P]),
    "pas_last_launch_count": (C.c_int, [_P]),
    "pas_debug_scores": (C.c_int, [_P, _P, C.c_int, C.c_int64, _P, _P]),
    "pas_debug_k2_schedule": (C.c_int, [C.c_int64, C.c_int64, C.c_int, C.c_int64, _P]),
    "pas_debug_qhat": (C.c_int, [_P, _P, C.c_int64, _P]),
    "pas_debug_store_rows": (C.c_int, [_P, C.c_int64, C.c_int64, _P, _P]),
}
for _name, (_res, _args) in _SIG.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIG)


def _check(ctx, status: int):
    if status != PAS_OK:
        msg = lib.pas_last_error(ctx)
        raise PasError(status, msg.decode() if msg else "")


# ----------------------------------------------------------------------------------------------
# same-name wrappers (raise PasError instead of returning a status)
# ----------------------------------------------------------------------------------------------
def pas_version() -> str:
    return lib.pas_version().decode()


def pas_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(PAS_NCCL_ID_BYTES)
    _check(None, lib.pas_nccl_unique_id(buf))
    return buf.raw


def pas_create(d=768, topk=8, max_batch=4096, max_rows_per_rank=1 << 20, device=0, rank=0, world=1,
               nccl_id: bytes | None = None, seed=0x5EED2502):
    cfg = PasConfig(d, topk, max_batch, max_rows_per_rank, device, rank, world, None, seed)
    keep = None
    if nccl_id is not None:
        keep = C.create_string_buffer(bytes(nccl_id), PAS_NCCL_ID_BYTES)
        cfg.nccl_id = C.cast(keep, C.c_void_p)
    ctx = _P()
    _check(None, lib.pas_create(C.byref(ctx), C.byref(cfg)))
    _CTX_D[ctx.value] = d
    return ctx


def pas_destroy(ctx):
    _CTX_D.pop(ctx.value, None)
    _check(None, lib.pas_destroy(ctx))


def _stream(stream):
    if stream is None:
        import torch
        return _P(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return _P(stream)
    return _P(stream.cuda_stream)


_CTX_D: dict = {}   # embedding width d of each live context (argument checks only)


def _rows(ctx, t, device=True):
    """Embedding rows [n, d] as the C side reads them: contiguous (row stride d), width d, on the
    device (or the host for pas_route_batch_host).  Raises instead of letting K1 read out of bounds."""
    d = _CTX_D.get(ctx.value if isinstance(ctx, _P) else ctx)
    if t.dim() != 2 or (d is not None and t.shape[1] != d):
        raise ValueError(f"embeddings must be [n, {d}], got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError("embeddings must be contiguous (row-major, stride d)")
    if t.is_cuda != device:
        raise ValueError("embeddings must be a CUDA tensor" if device else "embeddings must be a host tensor")
    return _P(t.data_ptr())


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return PAS_F32
    if t.dtype == torch.bfloat16:
        return PAS_BF16
    raise TypeError(f"embeddings must be float32 or bfloat16, got {t.dtype}")


def pas_cache_load(ctx, rows, stream=None) -> int:
    """rows: contiguous CUDA tensor [M, d] (float32 / bfloat16).  Returns the first global id."""
    first = C.c_int64(0)
    _check(ctx, lib.pas_cache_load(ctx, _rows(ctx, rows), _dtype_code(rows), rows.shape[0],
                                   C.byref(first), _stream(stream)))
    return first.value


def pas_cache_clear(ctx):
    _check(ctx, lib.pas_cache_clear(ctx))


def pas_cache_size(ctx):
    g, l_ = C.c_int64(0), C.c_int64(0)
    _check(ctx, lib.pas_cache_size(ctx, C.byref(g), C.byref(l_)))
    return g.value, l_.value


def pas_set_bands(ctx, K_levels, thresholds):
    nK = len(K_levels)
    kl = (C.c_int32 * nK)(*K_levels)
    th = (C.c_float * max(1, nK - 1))(*thresholds)
    _check(ctx, lib.pas_set_bands(ctx, kl, nK, th))


def pas_set_degradation(ctx, c):
    arr = (C.c_double * len(c))(*c)
    _check(ctx, lib.pas_set_degradation(ctx, arr, len(c)))


def pas_set_fractions(ctx, F, instance_level, bstar=4, mode=PAS_GREEDY):
    Fa = (C.c_double * len(F))(*F)
    il = (C.c_int32 * len(instance_level))(*instance_level)
    _check(ctx, lib.pas_set_fractions(ctx, Fa, il, len(instance_level), bstar, mode))


PAS_COLL_FOLDED, PAS_COLL_EXPLICIT = 0, 1


def pas_set_collectives(ctx, mode):
    _check(ctx, lib.pas_set_collectives(ctx, mode))


def pas_set_graph(ctx, on=True):
    _check(ctx, lib.pas_set_graph(ctx, 1 if on else 0))


def pas_stage_ring(ctx, slots):
    _check(ctx, lib.pas_stage_ring(ctx, slots))


def pas_stage_ring_read(ctx, n) -> list:
    """Per-batch stage times (ms) of the last <= n batches, oldest first: lists of 7 floats."""
    buf = (C.c_float * (7 * max(1, n)))()
    got = C.c_int(0)
    _check(ctx, lib.pas_stage_ring_read(ctx, n, buf, C.byref(got)))
    return [list(buf[7 * b:7 * b + 7]) for b in range(got.value)]


def pas_set_seed(ctx, seed, batch_seq=0):
    _check(ctx, lib.pas_set_seed(ctx, seed, batch_seq))


def pas_cache_insert(ctx, rows, gids_out=None, stream=None):
    _check(ctx, lib.pas_cache_insert(ctx, _rows(ctx, rows), _dtype_code(rows), rows.shape[0],
                                     _P(gids_out.data_ptr()) if gids_out is not None else None, _stream(stream)))


def pas_cache_insert_vanilla(ctx, emb, K_prime, gids_by_prompt=None, stream=None) -> int:
    n = C.c_int64(0)
    _check(ctx, lib.pas_cache_insert_vanilla(ctx, _rows(ctx, emb), _dtype_code(emb), emb.shape[0],
                                             _P(K_prime.data_ptr()),
                                             _P(gids_by_prompt.data_ptr()) if gids_by_prompt is not None else None,
                                             C.byref(n), _stream(stream)))
    return n.value


def pas_cache_stamps(ctx, out, stream=None):
    _check(ctx, lib.pas_cache_stamps(ctx, _P(out.data_ptr()), out.numel(), _stream(stream)))


def pas_set_forecast(ctx, window, replan_every=1):
    _check(ctx, lib.pas_set_forecast(ctx, window, replan_every))


def pas_set_dispatcher(ctx, service_us, timeout_us=250_000):
    """service_us: per-instance batch service times (us), or None to turn the dispatcher off."""
    if service_us is None:
        _check(ctx, lib.pas_set_dispatcher(ctx, None, 0, 0))
        return
    arr = (C.c_int64 * len(service_us))(*service_us)
    _check(ctx, lib.pas_set_dispatcher(ctx, arr, len(service_us), timeout_us))


def pas_set_clock(ctx, now_us):
    _check(ctx, lib.pas_set_clock(ctx, now_us))


def pas_set_load(ctx, lambda_rps, bstar_high) -> int:
    m = C.c_int(0)
    _check(ctx, lib.pas_set_load(ctx, float(lambda_rps), bstar_high, C.byref(m)))
    return m.value


def pas_dispatcher_state(ctx, W) -> dict:
    arrs = [(C.c_int64 * W)() for _ in range(4)]
    _check(ctx, lib.pas_dispatcher_state(ctx, *arrs))
    return dict(queue=list(arrs[0]), busy_until=list(arrs[1]), fired_prompts=list(arrs[2]),
                fired_batches=list(arrs[3]))


def pas_solve_assignment(ctx, W, lambda_rps, H, service_us, bstar) -> dict:
    """H: per-level forecast, or None for the f1 predictor window."""
    a = PasAssignment()
    Ha = None if H is None else (C.c_double * len(H))(*H)
    sv = (C.c_int64 * len(service_us))(*service_us)
    _check(ctx, lib.pas_solve_assignment(ctx, W, float(lambda_rps), Ha, sv, bstar, C.byref(a)))
    nK = a.nK
    return dict(n=list(a.n[:nK]), F=list(a.F[:nK]), F_route=list(a.F_route[:nK]), H=list(a.H[:nK]),
                S=a.served, q=a.quality, instance_level=list(a.instance_level[:W]),
                candidates=a.candidates, solve_ms=a.solve_ms)


def _ptr(t):
    return None if t is None else t.data_ptr()


def make_out(**arrays) -> PasRouteOut:
    return PasRouteOut(*[_ptr(arrays.get(f)) for f, _ in PasRouteOut._fields_])


def pas_route_batch(ctx, emb, out: dict, stream=None):
    o = make_out(**out)
    _check(ctx, lib.pas_route_batch(ctx, _rows(ctx, emb), _dtype_code(emb), emb.shape[0], C.byref(o),
                                    _stream(stream)))


def pas_route_batch_host(ctx, emb, out: dict, stream=None):
    """emb: CPU tensor (pinned for speed); out: dict of CPU tensors."""
    o = make_out(**out)
    _check(ctx, lib.pas_route_batch_host(ctx, _rows(ctx, emb, device=False), _dtype_code(emb), emb.shape[0],
                                         C.byref(o), _stream(stream)))


def pas_route_batch_host_async(ctx, emb, out: dict, stream=None):
    """Pipelined host-buffer routing (include/pas.h): returns before the batch is done; emb and the
    out tensors (CPU, pinned) must stay alive and untouched until pas_route_host_end + a stream sync."""
    o = make_out(**out)
    _check(ctx, lib.pas_route_batch_host_async(ctx, _rows(ctx, emb, device=False), _dtype_code(emb), emb.shape[0],
                                               C.byref(o), _stream(stream)))


def pas_route_host_begin(ctx, stream=None):
    _check(ctx, lib.pas_route_host_begin(ctx, _stream(stream)))


def pas_route_host_end(ctx, stream=None):
    _check(ctx, lib.pas_route_host_end(ctx, _stream(stream)))


def pas_route_local(ctx, emb, cand, stream=None):
    """cand: CUDA int64/float tensor with N*topk 8-byte elements (pairs {float score, int32 gid})."""
    _check(ctx, lib.pas_route_local(ctx, _rows(ctx, emb), _dtype_code(emb), emb.shape[0],
                                    _P(cand.data_ptr()), _stream(stream)))


def pas_route_from_candidates(ctx, cand, S, N, out: dict, stream=None):
    o = make_out(**out)
    _check(ctx, lib.pas_route_from_candidates(ctx, _P(cand.data_ptr()), S, N, C.byref(o), _stream(stream)))


def pas_plan_stats(ctx) -> dict:
    s = PasStats()
    _check(ctx, lib.pas_plan_stats(ctx, C.byref(s)))
    nK, W = s.nK, s.W
    return dict(nK=nK, W=W, N=s.N, h=list(s.h[:nK]), f=list(s.f[:nK]),
                x=[list(s.x[i][:nK]) for i in range(nK)], D_Q=s.D_Q, D_Q_LP=s.D_Q_LP,
                plan_solver_iters=s.plan_solver_iters,
                n_redirected=s.n_redirected, n_upgraded=s.n_upgraded, n_downgraded=s.n_downgraded,
                n_invalid=s.n_invalid, n_near_top1=s.n_near_top1, n_near_threshold=s.n_near_threshold,
                bucket_count=list(s.bucket_count[:W]), stage_ms=list(s.stage_ms),
                forecast=s.forecast, fc_replanned=s.fc_replanned, fc_plan_n=s.fc_plan_n,
                fc_plan_counts=list(s.fc_plan_counts[:nK]), fc_window_n=s.fc_window_n,
                fc_l2_error=s.fc_l2_error, n_unforecast=s.n_unforecast,
                fc_Hc=list(s.fc_Hc[:nK + 1]), fc_Fc=list(s.fc_Fc[:nK + 1]),
                dispatcher=s.dispatcher, now_us=s.now_us, queue_len=list(s.queue_len[:W]),
                busy_until_us=list(s.busy_until_us[:W]), fired_prompts=list(s.fired_prompts[:W]),
                fired_batches=list(s.fired_batches[:W]), k2_ranges=s.k2_ranges,
                k2_chunk_tiles=s.k2_chunk_tiles, k2_chunk_steps=s.k2_chunk_steps, k6_fallback=s.k6_fallback)


def pas_last_launch_count(ctx) -> int:
    return lib.pas_last_launch_count(ctx)


def pas_debug_k2_schedule(N, M_local, d=768, max_batch=None) -> dict:
    """K2's schedule for a batch (host logic, no device): R, T (0 = static), CS, MTg, pair, MT, NT."""
    out = (C.c_int * 9)()
    st = lib.pas_debug_k2_schedule(N, M_local, d, N if max_batch is None else max_batch, out)
    if st != PAS_OK:
        raise PasError(st, "pas_debug_k2_schedule: bad arguments")
    return dict(zip(("R", "T", "CS", "MTg", "pair", "MT", "NT", "cand_cap", "tile_rows"), list(out)))


def pas_debug_qhat(ctx, out, stream=None):
    """out: CUDA bfloat16 / int16 tensor [N, d] receiving the last batch's quantised prompts."""
    assert out.is_cuda and out.is_contiguous() and out.element_size() == 2
    _check(ctx, lib.pas_debug_qhat(ctx, _P(out.data_ptr()), out.shape[0], _stream(stream)))


def pas_debug_store_rows(ctx, first_local_row, out, stream=None):
    """out: CUDA bfloat16 / int16 tensor [n, d] receiving this rank's store rows from first_local_row."""
    assert out.is_cuda and out.is_contiguous() and out.element_size() == 2
    _check(ctx, lib.pas_debug_store_rows(ctx, first_local_row, out.shape[0], _P(out.data_ptr()), _stream(stream)))


def pas_debug_scores(ctx, emb, scores, stream=None):
    _check(ctx, lib.pas_debug_scores(ctx, _rows(ctx, emb), _dtype_code(emb), emb.shape[0],
                                     _P(scores.data_ptr()), _stream(stream)))


# ----------------------------------------------------------------------------------------------
# convenience: a router object owning its output tensors
# ----------------------------------------------------------------------------------------------
class Router:
    """Owns one libpas context on ``device`` and reusable output tensors (argument marshalling only)."""

    def __init__(self, d=768, topk=8, max_batch=4096, max_rows_per_rank=1 << 20, device=0, rank=0,
                 world=1, nccl_id=None, seed=0x5EED2502):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.topk = topk
        self.W = 0
        self.ctx = pas_create(d, topk, max_batch, max_rows_per_rank, device, rank, world, nccl_id, seed)
        self._out = None

    def close(self):
        if self.ctx:
            pas_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_cache(self, rows, stream=None) -> int:
        return pas_cache_load(self.ctx, rows, stream)

    def set_bands(self, K_levels, thresholds):
        pas_set_bands(self.ctx, K_levels, thresholds)

    def set_degradation(self, c):
        pas_set_degradation(self.ctx, c)

    def set_fractions(self, F, instance_level, bstar=4, mode=PAS_GREEDY):
        pas_set_fractions(self.ctx, F, instance_level, bstar, mode)
        self.W = len(instance_level)

    def set_seed(self, seed, batch_seq=0):
        pas_set_seed(self.ctx, seed, batch_seq)

    def insert(self, rows, gids_out=None, stream=None):
        pas_cache_insert(self.ctx, rows, gids_out, stream)

    def insert_vanilla(self, emb, K_prime, gids_by_prompt=None, stream=None) -> int:
        return pas_cache_insert_vanilla(self.ctx, emb, K_prime, gids_by_prompt, stream)

    def set_forecast(self, window, replan_every=1):
        pas_set_forecast(self.ctx, window, replan_every)

    def solve_assignment(self, W, lambda_rps, H, service_us, bstar) -> dict:
        return pas_solve_assignment(self.ctx, W, lambda_rps, H, service_us, bstar)

    def set_dispatcher(self, service_us, timeout_us=250_000):
        pas_set_dispatcher(self.ctx, service_us, timeout_us)

    def set_clock(self, now_us):
        pas_set_clock(self.ctx, now_us)

    def set_load(self, lambda_rps, bstar_high) -> int:
        return pas_set_load(self.ctx, lambda_rps, bstar_high)

    def dispatcher_state(self) -> dict:
        return pas_dispatcher_state(self.ctx, self.W)

    def alloc_out(self, N, optional=True, device=None):
        t = self.torch
        dev = self.device if device is None else device
        i32 = dict(dtype=t.int32, device=dev)
        out = dict(K=t.empty(N, **i32), K_prime=t.empty(N, **i32), instance=t.empty(N, **i32),
                   slot=t.empty(N, **i32))
        if optional:
            out.update(topk_id=t.empty(N * self.topk, **i32),
                       topk_score=t.empty(N * self.topk, dtype=t.float32, device=dev),
                       flags=t.empty(N, dtype=t.uint8, device=dev),
                       bucket_offsets=t.empty(PAS_MAX_INSTANCES + 1, **i32),
                       bucket_prompts=t.empty(N, **i32))
        return out

    def route(self, emb, out=None, stream=None):
        if out is None:
            out = self.alloc_out(emb.shape[0])
        pas_route_batch(self.ctx, emb, out, stream)
        return out

    def stats(self):
        return pas_plan_stats(self.ctx)
