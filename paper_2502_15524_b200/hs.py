"""ctypes binding of libhs.so (include/hs.h, include/hs_kernels.h) — argument marshalling only.

Every step of the path runs in the library's CUDA kernels / copy engines; this module only
converts Python values to C structs and pointers.  There is no fallback: if libhs.so is not
built, importing raises (build it with ``python -m paper_2502_15524_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libhs.so")
if os.environ.get("HS_LIB_VARIANT"):  # same-box A/B of two builds (tools/build_variant.py); in-tree only
    SO = os.path.join(HERE, os.path.basename(os.environ["HS_LIB_VARIANT"]))

HS_MAX_STAGES = 8
HS_MAX_LAYERS = 128
STATUS = {0: "HS_OK", 1: "HS_E_INVAL", 2: "HS_E_CUDA", 3: "HS_E_OOM", 4: "HS_E_INFEASIBLE",
          5: "HS_E_STATE", 6: "HS_E_PEER", 7: "HS_E_TIMEOUT"}


class HsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class ModelCfg(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("max_seq", C.c_int32), ("rms_eps", C.c_float),
                ("rope_theta", C.c_float)]


class ImageHeader(C.Structure):
    _fields_ = [("magic", C.c_uint64), ("version", C.c_uint32), ("gu_interleave", C.c_uint32),
                ("cfg", ModelCfg), ("total_bytes", C.c_uint64), ("embed_off", C.c_uint64),
                ("embed_bytes", C.c_uint64), ("layer_off", C.c_uint64 * HS_MAX_LAYERS),
                ("layer_bytes", C.c_uint64), ("t_attn_norm", C.c_uint64), ("t_wqkv", C.c_uint64),
                ("t_wo", C.c_uint64), ("t_ffn_norm", C.c_uint64), ("t_wgu", C.c_uint64),
                ("t_wd", C.c_uint64), ("final_off", C.c_uint64), ("final_bytes", C.c_uint64),
                ("t_final_norm", C.c_uint64), ("t_lm_head", C.c_uint64), ("param_bytes", C.c_uint64)]


class Image(C.Structure):
    _fields_ = [("header", C.POINTER(ImageHeader)), ("data", C.c_void_p),
                ("data_offset", C.c_uint64), ("data_bytes", C.c_uint64), ("fetched_end", C.c_void_p)]


class Gpu(C.Structure):
    _fields_ = [("device", C.c_int32), ("h2d_gbps", C.c_double), ("link_group", C.c_int32),
                ("free_bytes", C.c_uint64), ("n_workers", C.c_int32)]


class Slo(C.Structure):
    _fields_ = [("t_prefill_s", C.c_double), ("t_decode_s", C.c_double), ("t_hop_s", C.c_double),
                ("slo_ttft_s", C.c_double), ("slo_tpot_s", C.c_double), ("max_pp", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [("pp", C.c_int32), ("device", C.c_int32 * HS_MAX_STAGES),
                ("layer_begin", C.c_int32 * HS_MAX_STAGES), ("layer_end", C.c_int32 * HS_MAX_STAGES),
                ("stage_bytes", C.c_uint64 * HS_MAX_STAGES), ("slice_begin", C.c_uint64 * HS_MAX_STAGES),
                ("slice_end", C.c_uint64 * HS_MAX_STAGES), ("full_memory", C.c_int32 * HS_MAX_STAGES),
                ("pred_ttft_s", C.c_double)]

    def as_dict(self):
        n = self.pp
        return dict(pp=n, device=list(self.device[:n]),
                    ranges=[(self.layer_begin[k], self.layer_end[k]) for k in range(n)],
                    stage_bytes=list(self.stage_bytes[:n]),
                    slices=[(self.slice_begin[k], self.slice_end[k]) for k in range(n)],
                    full_memory=list(self.full_memory[:n]), pred_ttft_s=self.pred_ttft_s)


class KvCfg(C.Structure):
    _fields_ = [("block_tokens", C.c_int32), ("num_blocks", C.c_int32), ("max_seqs", C.c_int32),
                ("max_tokens", C.c_int32)]


ALLGATHER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
BARRIER = C.CFUNCTYPE(C.c_int32, C.c_void_p)


class Comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("ctx", C.c_void_p),
                ("allgather", ALLGATHER), ("barrier", BARRIER)]


class LoadStats(C.Structure):
    _fields_ = [("bytes", C.c_uint64), ("load_ms", C.c_float), ("layers_ready", C.c_int32),
                ("done", C.c_int32)]


class StageTiming(C.Structure):
    _fields_ = [("load_ms", C.c_float), ("call_ms", C.c_float), ("since_load_ms", C.c_float)]


class ProfEntry(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("count", C.c_uint64), ("ms", C.c_double), ("bytes", C.c_double),
                ("flops", C.c_double)]


class ConsolidateStats(C.Structure):
    _fields_ = [("weight_bytes", C.c_uint64), ("kv_bytes", C.c_uint64), ("seconds", C.c_double),
                ("pause_seconds", C.c_double), ("weight_bytes_host", C.c_uint64),
                ("weight_bytes_background", C.c_uint64)]


# exported symbols (include/hs.h + include/hs_kernels.h); tests check every one is present
SYMBOLS = ["hs_image_layout", "hs_plan_stages", "hs_predict_ttft_eq1", "hs_predict_tpot_eq2",
           "hs_predict_ttft_eq5", "hs_group_create", "hs_load_stage_async", "hs_stage_load_stats",
           "hs_prefill", "hs_decode_step", "hs_release_seq", "hs_consolidate", "hs_group_destroy",
           "hs_last_error", "hs_group_info", "hs_debug_read_kv", "hs_debug_read_weights",
           "hs_debug_poison_weights", "hs_debug_launch_count", "hs_stage_timing_get", "hs_profile_enable",
           "hs_profile_read", "hs_debug_comm_selftest",
           "hs_k_gemm", "hs_k_rmsnorm", "hs_k_rope_kv", "hs_k_attention", "hs_k_argmax", "hs_k_embed",
           "hs_k_span_copy", "hs_debug_gemm_trace", "hs_debug_dstack_trace", "hs_debug_dstack_diag", "hs_plan_auto", "hs_links_create", "hs_links_admit",
           "hs_links_settle", "hs_links_complete", "hs_links_pending", "hs_links_destroy",
           "hs_load_background_async", "hs_scale_up", "hs_release_peer_memory", "hs_debug_capture",
           "hs_debug_read_hidden", "hs_debug_set_prefill_chunking", "hs_prefetch_start", "hs_prefetch_wait",
           "hs_prefetch_destroy", "hs_decode_steps", "hs_place_cold_start", "hs_pull_background_async"]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO):
        raise ImportError(f"{SO} is missing: build the CUDA library first "
                          "(python -m paper_2502_15524_b200.build); there is no fallback path")
    L = C.CDLL(SO)
    P, I32, U64, VP = C.POINTER, C.c_int32, C.c_uint64, C.c_void_p
    L.hs_last_error.restype = C.c_char_p
    L.hs_image_layout.argtypes = [P(ModelCfg), P(ImageHeader)]
    L.hs_plan_stages.argtypes = [P(ModelCfg), P(Gpu), I32, I32, I32, C.c_double, C.c_double, P(Plan)]
    for f in ("hs_predict_ttft_eq1",):
        getattr(L, f).restype = C.c_double
        getattr(L, f).argtypes = [C.c_double, C.c_double, I32, I32, P(C.c_double), P(C.c_double),
                                  C.c_double, C.c_double]
    L.hs_predict_tpot_eq2.restype = C.c_double
    L.hs_predict_tpot_eq2.argtypes = [C.c_double, I32, I32, C.c_double]
    L.hs_predict_ttft_eq5.restype = C.c_double
    L.hs_predict_ttft_eq5.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, I32, I32,
                                      P(C.c_double), P(C.c_double), C.c_double, C.c_double]
    L.hs_group_create.argtypes = [P(ModelCfg), P(Plan), P(Image), P(Image), P(KvCfg), P(Comm), P(VP)]
    L.hs_load_stage_async.argtypes = [VP, I32, U64]
    L.hs_stage_load_stats.argtypes = [VP, I32, I32, P(LoadStats)]
    L.hs_prefill.argtypes = [VP, I32, VP, VP, VP, VP, VP]
    L.hs_decode_step.argtypes = [VP, I32, VP, VP, VP, VP]
    L.hs_release_seq.argtypes = [VP, C.c_int64]
    L.hs_consolidate.argtypes = [VP, I32, P(ConsolidateStats)]
    L.hs_group_destroy.argtypes = [VP]
    L.hs_release_peer_memory.argtypes = [VP]
    L.hs_group_info.argtypes = [VP, P(I32), P(I32)]
    L.hs_debug_read_kv.argtypes = [VP, C.c_int64, I32, I32, I32, VP]
    L.hs_debug_read_weights.argtypes = [VP, I32, U64, U64, VP]
    L.hs_debug_poison_weights.argtypes = [VP, I32]
    L.hs_debug_launch_count.argtypes = [VP, P(U64)]
    L.hs_stage_timing_get.argtypes = [VP, I32, P(StageTiming)]
    L.hs_profile_enable.argtypes = [VP, I32]
    L.hs_profile_read.argtypes = [VP, P(ProfEntry), I32, P(I32), I32]
    L.hs_debug_comm_selftest.argtypes = [P(Comm)]
    L.hs_k_gemm.argtypes = [VP, I32, I32, VP, I32, I32, I32, VP, I32, VP, I32, VP, U64, VP]
    L.hs_k_rmsnorm.argtypes = [VP, VP, VP, VP, I32, I32, C.c_float, VP]
    L.hs_k_rope_kv.argtypes = [VP, VP, VP, VP, VP, VP, I32, I32, I32, VP]
    L.hs_k_attention.argtypes = [VP, VP, VP, I32, I32, I32, VP, I32, VP, I32, I32, I32, VP, VP]
    L.hs_k_argmax.argtypes = [VP, I32, I32, VP, VP]
    L.hs_k_embed.argtypes = [VP, VP, VP, I32, I32, VP]
    L.hs_k_span_copy.argtypes = [VP, VP, I32, U64, VP]
    L.hs_debug_gemm_trace.argtypes = [I32, VP, I32]
    L.hs_debug_dstack_trace.argtypes = [I32, VP, C.c_int64]
    L.hs_debug_dstack_diag.argtypes = [I32]
    L.hs_debug_dstack_diag.restype = I32
    L.hs_plan_auto.argtypes = [P(ModelCfg), P(Gpu), I32, P(Slo), P(Plan), P(I32)]
    L.hs_links_create.argtypes = [I32, P(C.c_double), P(VP)]
    L.hs_links_admit.argtypes = [VP, I32, C.c_double, C.c_double, C.c_double, P(I32), P(C.c_int64)]
    L.hs_links_settle.argtypes = [VP, I32, C.c_double]
    L.hs_links_complete.argtypes = [VP, I32, C.c_int64, C.c_double]
    L.hs_links_pending.argtypes = [VP, I32, I32, P(I32), P(C.c_double), P(C.c_int64)]
    L.hs_links_destroy.argtypes = [VP]
    L.hs_load_background_async.argtypes = [VP, I32, U64]
    L.hs_pull_background_async.argtypes = [VP, I32, U64]
    L.hs_scale_up.argtypes = [VP, P(I32), I32, P(VP), P(ConsolidateStats)]
    L.hs_debug_capture.argtypes = [VP, I32]
    L.hs_debug_read_hidden.argtypes = [VP, I32, I32, I32, VP]
    L.hs_debug_set_prefill_chunking.argtypes = [VP, I32, I32]
    L.hs_prefetch_start.argtypes = [C.c_char_p, U64, VP, U64, U64, C.c_double, VP, P(VP)]
    L.hs_prefetch_wait.argtypes = [VP, P(U64), P(C.c_double)]
    L.hs_prefetch_destroy.argtypes = [VP]
    L.hs_decode_steps.argtypes = [VP, I32, VP, VP, I32, I32, VP]
    L.hs_place_cold_start.argtypes = [P(ModelCfg), P(Gpu), I32, VP, C.c_double, C.c_double, I32, P(Plan),
                                      P(C.c_double), P(I32), P(C.c_int64)]
    _lib = L
    return L


def check(code):
    if code != 0:
        msg = lib().hs_last_error().decode()
        if code == 2:  # HS_E_CUDA: name the decode-stack wait that trapped, if one did
            lib().hs_debug_dstack_diag(1)
        raise HsError(code, msg)


def model_cfg(cfg: dict) -> ModelCfg:
    return ModelCfg(**{k: cfg[k] for k, _ in ModelCfg._fields_})


def image_layout(cfg: dict) -> ImageHeader:
    h = ImageHeader()
    c = model_cfg(cfg)
    check(lib().hs_image_layout(C.byref(c), C.byref(h)))
    return h


def _gpus(gpus):
    return (Gpu * len(gpus))(*[Gpu(g["device"], g["h2d_gbps"], g.get("link_group", 0), g["free_bytes"],
                                   g.get("n_workers", 0)) for g in gpus])


def plan_auto(cfg: dict, gpus, t_prefill_s, t_decode_s, t_hop_s, slo_ttft_s, slo_tpot_s, max_pp=4):
    """Algorithm 1: returns (plan, sharing, feasible)."""
    out, sh = Plan(), C.c_int32()
    c = model_cfg(cfg)
    slo = Slo(t_prefill_s, t_decode_s, t_hop_s, slo_ttft_s, slo_tpot_s, max_pp)
    r = lib().hs_plan_auto(C.byref(c), _gpus(gpus), len(gpus), C.byref(slo), C.byref(out), C.byref(sh))
    if r not in (0, 4):
        check(r)
    return out, sh.value, r == 0


class Links:
    """Eq. 3 / Eq. 4 contention registry over host-link groups (hs_links_*)."""

    def __init__(self, group_bytes_per_s):
        arr = (C.c_double * len(group_bytes_per_s))(*group_bytes_per_s)
        self.h = C.c_void_p()
        check(lib().hs_links_create(len(group_bytes_per_s), arr, C.byref(self.h)))

    def admit(self, group, pending, deadline, now):
        acc, wid = C.c_int32(), C.c_int64()
        check(lib().hs_links_admit(self.h, group, pending, deadline, now, C.byref(acc), C.byref(wid)))
        return bool(acc.value), wid.value

    def settle(self, group, now):
        check(lib().hs_links_settle(self.h, group, now))

    def complete(self, group, wid, now):
        check(lib().hs_links_complete(self.h, group, wid, now))

    def pending(self, group):
        n = C.c_int32()
        check(lib().hs_links_pending(self.h, group, 0, C.byref(n), None, None))
        pend = (C.c_double * max(n.value, 1))()
        ids = (C.c_int64 * max(n.value, 1))()
        check(lib().hs_links_pending(self.h, group, n.value, C.byref(n), pend, ids))
        return {ids[i]: pend[i] for i in range(n.value)}

    def place(self, cfg: dict, gpus, now: float, slo_ttft_s: float, max_pp: int = 4):
        """hs_place_cold_start: (plan, predicted TTFT s, admitted, worker ids)."""
        out, pred, ok = Plan(), C.c_double(), C.c_int32()
        ids = (C.c_int64 * HS_MAX_STAGES)()
        c = model_cfg(cfg)
        check(lib().hs_place_cold_start(C.byref(c), _gpus(gpus), len(gpus), self.h, now, slo_ttft_s, max_pp,
                                        C.byref(out), C.byref(pred), C.byref(ok), ids))
        return out, pred.value, bool(ok.value), list(ids[:out.pp])

    def __del__(self):
        try:
            lib().hs_links_destroy(self.h)
        except Exception:  # noqa
            pass


def plan_stages(cfg: dict, gpus, pp: int, full_memory_stages: int = 1, t_prefill_s: float = 0.0,
                t_hop_s: float = 0.0) -> Plan:
    arr = _gpus(gpus)
    out = Plan()
    c = model_cfg(cfg)
    check(lib().hs_plan_stages(C.byref(c), arr, len(gpus), pp, full_memory_stages, t_prefill_s, t_hop_s, C.byref(out)))
    return out


def predict_ttft_eq1(t_c, M, s, w, b, p, t_p, t_n):
    D = C.c_double * s
    return lib().hs_predict_ttft_eq1(t_c, M, s, w, D(*b), D(*p), t_p, t_n)


def predict_tpot_eq2(t_d, s, w, t_n):
    return lib().hs_predict_tpot_eq2(t_d, s, w, t_n)


def predict_ttft_eq5(t_cc, t_cu, t_l, M, s, w, b, p, t_p, t_n):
    D = C.c_double * s
    return lib().hs_predict_ttft_eq5(t_cc, t_cu, t_l, M, s, w, D(*b), D(*p), t_p, t_n)


class HostImage:
    """A (slice of a) host weight image in pinned memory, filled by the caller's generator.
    Holds a torch pinned tensor (torch = plumbing for host/device memory)."""

    def __init__(self, header: ImageHeader, begin: int, end: int):
        import torch
        self.header = header
        self.begin, self.end = begin, end
        self.buf = torch.empty(end - begin, dtype=torch.uint8, pin_memory=True)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def c_image(self) -> Image:
        wm = C.c_void_p(self.watermark.data_ptr()) if getattr(self, "watermark", None) is not None else None
        return Image(C.pointer(self.header), C.c_void_p(self.ptr), self.begin, self.end - self.begin, wm)

    def prefetch_from(self, path: str, chunk_bytes: int = 0, max_gbps: float = 0.0) -> "Prefetch":
        """Starts the model prefetcher filling this image from `path` (the image's byte layout)
        and attaches its 8-byte fetched-end watermark: create the group afterwards."""
        import torch
        self.watermark = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        return Prefetch(path, self.begin, self.ptr, self.end - self.begin, self.watermark.data_ptr(), chunk_bytes,
                        max_gbps)


class Prefetch:
    """hs_prefetch_*: the model prefetcher thread."""

    def __init__(self, path, file_offset, dst, nbytes, watermark_ptr, chunk_bytes=0, max_gbps=0.0):
        self.h = C.c_void_p()
        check(lib().hs_prefetch_start(path.encode(), file_offset, C.c_void_p(dst), nbytes, chunk_bytes, max_gbps,
                                      C.c_void_p(watermark_ptr), C.byref(self.h)))

    def wait(self):
        """Joins the prefetcher: (bytes fetched, seconds)."""
        n, t = C.c_uint64(), C.c_double()
        check(lib().hs_prefetch_wait(self.h, C.byref(n), C.byref(t)))
        return n.value, t.value

    def destroy(self):
        if self.h:
            lib().hs_prefetch_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        self.destroy()


class DistComm:
    """hs_comm callbacks over torch.distributed (gloo sub-group for byte exchange)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.pg = dist.new_group(backend="gloo")
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

        def _ag(ctx, send, nbytes, recv):
            try:
                import torch
                t = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8)
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(outs, t, group=self.pg)
                cat = torch.cat(outs).numpy().tobytes()
                C.memmove(recv, cat, len(cat))
                return 0
            except Exception:  # noqa
                return 1

        def _bar(ctx):
            try:
                dist.barrier(group=self.pg)
                return 0
            except Exception:  # noqa
                return 1

        self._ag, self._bar = ALLGATHER(_ag), BARRIER(_bar)
        self.c = Comm(self.rank, self.world, None, self._ag, self._bar)


def comm_selftest(comm: "DistComm"):
    check(lib().hs_debug_comm_selftest(C.byref(comm.c)))


class Group:
    """A pipeline-parallel worker group (hs_group)."""

    def __init__(self, cfg: dict, plan: Plan, image: HostImage | None = None, stage_images=None,
                 num_blocks: int = 256, max_seqs: int = 16, max_tokens: int = 1024, comm: DistComm | None = None):
        self.cfg = cfg
        self.plan = plan
        self._c = model_cfg(cfg)
        self._img = image.c_image() if image is not None else None
        self._keep = [image, stage_images]
        self._stage_imgs = None
        if stage_images is not None:
            arr = (Image * plan.pp)(*[si.c_image() if si is not None else Image() for si in stage_images])
            self._stage_imgs = arr
        self._kv = KvCfg(16, num_blocks, max_seqs, max_tokens)
        self._comm = comm
        self.h = C.c_void_p()
        check(lib().hs_group_create(C.byref(self._c), C.byref(plan), C.byref(self._img) if self._img else None,
                                    self._stage_imgs, C.byref(self._kv), C.byref(comm.c) if comm else None,
                                    C.byref(self.h)))

    def load_stage_async(self, stage: int = -1, chunk_bytes: int = 0):
        check(lib().hs_load_stage_async(self.h, stage, chunk_bytes))

    def load_background_async(self, target: int = 0, chunk_bytes: int = 0):
        check(lib().hs_load_background_async(self.h, target, chunk_bytes))

    def pull_background_async(self, target: int = 0, chunk_bytes: int = 0):
        """The target pulls the other stages' weight slices over NVLink in the background."""
        check(lib().hs_pull_background_async(self.h, target, chunk_bytes))

    def load_stats(self, stage: int, wait: bool = True) -> LoadStats:
        s = LoadStats()
        check(lib().hs_stage_load_stats(self.h, stage, 1 if wait else 0, C.byref(s)))
        return s

    def prefill(self, seq_ids, prompts, want_logits: bool = False):
        n = len(seq_ids)
        ids = np.asarray(seq_ids, dtype=np.int64)
        lens = np.asarray([len(p) for p in prompts], dtype=np.int32)
        toks = np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.int32) for p in prompts]))
        out = np.zeros(n, dtype=np.int32)
        logits = np.zeros((n, self.cfg["vocab"]), dtype=np.float32) if want_logits else None
        check(lib().hs_prefill(self.h, n, ids.ctypes.data, toks.ctypes.data, lens.ctypes.data, out.ctypes.data,
                               logits.ctypes.data if logits is not None else None))
        return out, logits

    def decode_step(self, seq_ids, in_tokens=None, want_logits: bool = False):
        n = len(seq_ids)
        ids = np.asarray(seq_ids, dtype=np.int64)
        tin = None if in_tokens is None else np.ascontiguousarray(np.asarray(in_tokens, dtype=np.int32))
        out = np.zeros(n, dtype=np.int32)
        logits = np.zeros((n, self.cfg["vocab"]), dtype=np.float32) if want_logits else None
        check(lib().hs_decode_step(self.h, n, ids.ctypes.data, tin.ctypes.data if tin is not None else None,
                                   out.ctypes.data, logits.ctypes.data if logits is not None else None))
        return out, logits

    def decode_steps(self, seq_ids, n_steps: int, n_micro: int = 1, in_tokens=None):
        """n_steps pipelined greedy steps with n_micro micro-batches; returns tokens [n_steps, n]."""
        n = len(seq_ids)
        ids = np.asarray(seq_ids, dtype=np.int64)
        tin = None if in_tokens is None else np.ascontiguousarray(np.asarray(in_tokens, dtype=np.int32))
        out = np.zeros((n_steps, n), dtype=np.int32)
        check(lib().hs_decode_steps(self.h, n, ids.ctypes.data, tin.ctypes.data if tin is not None else None, n_steps,
                                    n_micro, out.ctypes.data))
        return out

    def release_seq(self, seq_id: int):
        check(lib().hs_release_seq(self.h, seq_id))

    def consolidate(self, target: int = 0) -> ConsolidateStats:
        s = ConsolidateStats()
        check(lib().hs_consolidate(self.h, target, C.byref(s)))
        return s

    def release_peer_memory(self):
        """SPMD, collective: free the HBM consolidation released on the non-target ranks (after
        every rank has closed its peer mappings of it)."""
        check(lib().hs_release_peer_memory(self.h))

    def scale_up(self, seq_owner=None):
        """Every stage becomes a standalone endpoint; returns (list of Group, stats).  This group
        is emptied (destroy it).  The first decode of each endpoint must pass in_tokens."""
        pp = self.plan.pp
        outs = (C.c_void_p * pp)()
        st = ConsolidateStats()
        if seq_owner is not None:
            arr = (C.c_int32 * len(seq_owner))(*seq_owner)
            check(lib().hs_scale_up(self.h, arr, len(seq_owner), outs, C.byref(st)))
        else:
            check(lib().hs_scale_up(self.h, None, 0, outs, C.byref(st)))
        groups = []
        for i in range(pp if self._comm is None else 1):
            g = Group.__new__(Group)
            g.cfg, g.plan, g._c, g._img, g._keep, g._stage_imgs, g._kv, g._comm = \
                self.cfg, self.plan, self._c, self._img, self._keep, self._stage_imgs, self._kv, None
            g.h = C.c_void_p(outs[i])
            groups.append(g)
        return groups, st

    def info(self):
        pp, owned = C.c_int32(), C.c_int32()
        check(lib().hs_group_info(self.h, C.byref(pp), C.byref(owned)))
        return pp.value, owned.value

    def read_kv(self, seq_id: int, layer: int, pos0: int, n: int) -> np.ndarray:
        out = np.zeros((n, 2, self.cfg["n_heads"], self.cfg["head_dim"]), dtype=np.uint16)
        check(lib().hs_debug_read_kv(self.h, seq_id, layer, pos0, n, out.ctypes.data))
        return out

    def capture(self, on: bool = True):
        """Test-only: store every layer boundary's hidden rows of later calls (hs_debug_capture)."""
        check(lib().hs_debug_capture(self.h, 1 if on else 0))

    def read_hidden(self, boundary: int, row0: int = 0, n: int | None = None) -> np.ndarray:
        """bf16 bits [n, hidden] of layer boundary `boundary` of the latest call, call order."""
        if n is None:
            raise ValueError("pass the number of rows")
        out = np.zeros((n, self.cfg["hidden"]), dtype=np.uint16)
        check(lib().hs_debug_read_hidden(self.h, boundary, row0, n, out.ctypes.data))
        return out

    def set_prefill_chunking(self, min_chunk_tokens: int = 0, max_chunks: int = 0):
        check(lib().hs_debug_set_prefill_chunking(self.h, min_chunk_tokens, max_chunks))

    def read_weights(self, stage: int, off: int, nbytes: int) -> np.ndarray:
        out = np.empty(nbytes, dtype=np.uint8)
        check(lib().hs_debug_read_weights(self.h, stage, off, nbytes, out.ctypes.data))
        return out

    def poison(self, stage: int):
        check(lib().hs_debug_poison_weights(self.h, stage))

    def timing(self, stage: int) -> StageTiming:
        t = StageTiming()
        check(lib().hs_stage_timing_get(self.h, stage, C.byref(t)))
        return t

    def profile(self, on: bool):
        check(lib().hs_profile_enable(self.h, 1 if on else 0))

    def profile_read(self, reset: bool = True) -> dict:
        arr = (ProfEntry * 64)()
        n = C.c_int32()
        check(lib().hs_profile_read(self.h, arr, 64, C.byref(n), 1 if reset else 0))
        return {arr[i].name.decode(): dict(count=arr[i].count, ms=arr[i].ms, bytes=arr[i].bytes, flops=arr[i].flops)
                for i in range(min(n.value, 64))}

    @staticmethod
    def launch_count() -> int:
        v = C.c_uint64()
        check(lib().hs_debug_launch_count(None, C.byref(v)))
        return v.value

    def destroy(self):
        """Frees the group.  SPMD groups: collective, every rank must call it explicitly."""
        if self.h:
            h, self.h = self.h, C.c_void_p()
            check(lib().hs_group_destroy(h))

    def __del__(self):
        # local groups are freed on collection; an SPMD group's destroy is collective (it meets
        # the peers at a barrier) and must never run from a garbage collector on one rank only
        if getattr(self, "_comm", None) is not None:
            return
        try:
            self.destroy()
        except Exception:  # noqa
            pass


# ---------------------------------------------------------------- kernel entry points -------
def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def k_gemm(W, X, N, epi, out, resid=None, ws=None):
    M, K = W.shape
    ldo = out.shape[-1]
    check(lib().hs_k_gemm(_p(W), M, K, _p(X), X.shape[0], N, epi, _p(out), ldo, _p(resid),
                          resid.shape[-1] if resid is not None else 0, _p(ws),
                          ws.numel() * ws.element_size() if ws is not None else 0, _stream()))


def k_rmsnorm(x, w, y, eps, rows=None, T=None):
    T = T if T is not None else (rows.numel() if rows is not None else x.shape[0])
    check(lib().hs_k_rmsnorm(_p(x), _p(rows), _p(w), _p(y), T, x.shape[1], eps, _stream()))


def k_rope_kv(qkv, pos, slot, tab, q_out, pool, n_heads, head_dim):
    check(lib().hs_k_rope_kv(_p(qkv), _p(pos), _p(slot), _p(tab), _p(q_out), _p(pool), qkv.shape[0], n_heads,
                             head_dim, _stream()))


def k_attention(q, pool, seqs, max_nq, max_ctx, tables, o, n_heads, head_dim, decode, ws=None):
    check(lib().hs_k_attention(_p(q), _p(pool), _p(seqs), seqs.shape[0], max_nq, max_ctx, _p(tables),
                               tables.shape[1], _p(o), n_heads, head_dim, 1 if decode else 0, _p(ws), _stream()))


def k_argmax(logits, tokens):
    check(lib().hs_k_argmax(_p(logits), logits.shape[1], logits.shape[0], _p(tokens), _stream()))


def k_embed(tok, E, x):
    check(lib().hs_k_embed(_p(tok), _p(E), _p(x), tok.numel(), E.shape[1], _stream()))


def k_span_copy(src, dst, span_bytes):
    check(lib().hs_k_span_copy(_p(src), _p(dst), src.numel(), span_bytes, _stream()))


def dstack_trace(enable: bool, n_ctas: int = 0, n_layers: int = 0):
    """Per-CTA, per-layer phase stamps of the latest decode-stack launch ([n_ctas, n_layers, 32] ns)."""
    n = n_ctas * n_layers * 32
    extra = n_layers * 256 if n else 0
    out = np.zeros(max(n + extra, 1), dtype=np.uint64)
    check(lib().hs_debug_dstack_trace(1 if enable else 0, out.ctypes.data if n else None, n + extra))
    if not n:
        return None
    return out[:n].reshape(n_ctas, n_layers, 32), out[n:].reshape(n_layers, 256)


_probe = None


def probe_lib():
    """Test-only hardware probes (include/hs_probes.h), a separate library: never on a product path."""
    global _probe
    if _probe is None:
        lib()
        so = os.path.join(HERE, "libhs_probe.so")
        if not os.path.exists(so):
            raise ImportError(f"{so} is missing: build with python -m paper_2502_15524_b200.build")
        _probe = C.CDLL(so)
        _probe.hs_debug_tmem_a_gemm.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        _probe.hs_debug_stream_probe.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                                 C.POINTER(C.c_double)]
    return _probe


def stream_probe(layout: int, M: int, K: int, slots: int = 12, iters: int = 4) -> float:
    """Test-only: achieved GB/s streaming an [M, K] bf16 matrix in the decode stack's TMA pattern."""
    v = C.c_double()
    check(probe_lib().hs_debug_stream_probe(layout, M, K, slots, iters, C.byref(v)))
    return v.value


def tmem_a_gemm(A, B):
    """Test-only: (D with A from smem, D with A staged in TMEM), each [16, 128] fp32."""
    import torch
    K = A.shape[1]
    o1 = torch.empty(16, 128, dtype=torch.float32, device=A.device)
    o2 = torch.empty_like(o1)
    check(probe_lib().hs_debug_tmem_a_gemm(_p(A), _p(B), K, _p(o1), _p(o2)))
    return o1, o2


def gemm_trace(enable: bool, n_ctas: int = 0):
    out = np.zeros((max(n_ctas, 1), 8), dtype=np.uint64)
    check(lib().hs_debug_gemm_trace(1 if enable else 0, out.ctypes.data if n_ctas else None, n_ctas))
    return out[:n_ctas]
