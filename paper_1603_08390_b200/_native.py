"""ctypes bindings of the C ABI (include/genie/genie.h, include/genie/genie_synth.h).

The product path is libgenie_b200.so (hand-written sm_100a CUDA).  There is
no fallback: if the library is missing, importing the engine fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"
# GENIE_ENGINE_LIB selects an instrumented build (tools/phase_timers.py); default: the product library
ENGINE_LIB = Path(os.environ.get("GENIE_ENGINE_LIB", LIB_DIR / "libgenie_b200.so"))
SYNTH_LIB = LIB_DIR / "libgenie_synth.so"

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p

GENIE_OK = 0
GENIE_ERR_CONTRACT = 1
GENIE_ERR_DATA = 2
GENIE_ERR_INVARIANT = 3
GENIE_ERR_CUDA = 4
GENIE_ERR_NCCL = 5
GENIE_RETRY = 6
GENIE_FLAG_STAGE_EVENTS = 1
GENIE_FLAG_GRAPH = 2


class Entry(C.Structure):
    _fields_ = [("id", C.c_uint32), ("count", C.c_uint32)]


class Config(C.Structure):
    _fields_ = [
        ("selector", C.c_uint32),
        ("span_chunk", C.c_uint32),
        ("max_spans_per_task", C.c_uint32),
        ("tile_bytes", C.c_uint32),
        ("ctas_per_sm", C.c_uint32),
        ("flags", C.c_uint32),
    ]


class StageNs(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("lookup_ns", "match_ns", "select_ns", "merge_ns", "total_ns")]


class BatchStats(C.Structure):
    _fields_ = [
        (n, C.c_uint64)
        for n in ("counter_bytes", "gate_bytes", "table_bytes", "postings", "work_items", "fallback_tiles")
    ]


class LshConfig(C.Structure):
    _fields_ = [
        ("family", C.c_uint32),
        ("m", C.c_uint32),
        ("dims", C.c_uint32),
        ("rehash_domain", C.c_uint32),
        ("seed", C.c_uint64),
        ("w", C.c_double),
        ("bucket_count", C.c_uint32),
        ("rehash_pstable", C.c_int32),
        ("bucket_min", C.c_int64),
        ("sigma", C.c_double),
        ("precision", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


# name -> (restype, argtypes); every symbol declared in include/genie/genie.h
ENGINE_SYMBOLS = {
    "genie_config_default": (Config, []),
    "genie_index_build": (C.c_int, [C.c_uint32, u64p, u16p, u32p, C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "genie_mcix_parse": (C.c_int, [vp, C.c_uint64, u32p, u64p, u64p, u64p, u64p, u32p, C.c_char_p, C.c_size_t]),
    "genie_index_load_mcix": (C.c_int, [vp, C.c_uint64, C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "genie_mcix_serialize": (C.c_int, [C.c_uint32, C.c_uint64, u64p, u64p, u32p, C.c_uint32, vp, u64p, C.c_char_p,
                                       C.c_size_t]),
    "genie_index_create": (C.c_int, [C.c_uint32, C.c_uint64, u64p, u64p, u32p, u32p, C.c_uint32, C.c_int,
                                     C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "genie_index_create_shard": (C.c_int, [C.c_uint32, C.c_uint64, u64p, u64p, u32p, C.c_uint32, C.c_uint32,
                                           C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "genie_index_destroy": (None, [vp]),
    "genie_index_info": (None, [vp, u32p, u64p, u64p, u32p, C.POINTER(C.c_int)]),
    "genie_index_dim_stats": (C.c_int, [vp, u32p, C.c_char_p, C.c_size_t]),
    # host arrays as raw addresses (numpy .ctypes.data): the per-call argument
    # conversion is a few microseconds instead of ~4 us per pointer
    "genie_query_batch": (C.c_int, [vp, C.POINTER(Config), C.c_uint32, vp, vp, vp, vp, vp, vp,
                                    C.c_uint32, vp, vp, vp, vp, C.POINTER(StageNs),
                                    C.POINTER(BatchStats), C.c_char_p, C.c_size_t]),
    "genie_query_batch_device": (C.c_int, [vp, C.POINTER(Config), C.c_uint32, vp, vp, vp, vp, vp, vp,
                                           C.c_uint32, C.c_uint32, C.c_uint32, vp, vp, vp, vp, C.c_char_p,
                                           C.c_size_t]),
    "genie_query_status": (C.c_int, [vp, C.POINTER(BatchStats), C.c_char_p, C.c_size_t]),
    "genie_last_launch_count": (C.c_uint32, [vp]),
    "genie_graph_captures": (C.c_uint64, [vp]),
    "genie_last_stage_ns": (C.c_int, [vp, C.POINTER(StageNs), C.c_char_p, C.c_size_t]),
    "genie_debug_status": (C.c_int, [vp, u64p, C.c_uint32, C.c_char_p, C.c_size_t]),
    "genie_merge_topk_device": (C.c_int, [vp, C.c_uint32, C.c_uint32, vp, vp, C.c_uint32, vp, C.c_uint32,
                                          vp, vp, vp, vp, C.c_char_p, C.c_size_t]),
    "genie_merge_topk": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.POINTER(Entry), u32p, C.c_uint32, u32p,
                                   C.c_uint32, C.POINTER(Entry), u32p, u32p, C.c_char_p, C.c_size_t]),
    "genie_hash_results": (C.c_uint64, [C.c_uint32, u32p, u32p, u32p, C.c_uint32, C.POINTER(Entry)]),
    "genie_lsh_config_default": (LshConfig, []),
    "genie_lsh_sample": (C.c_int, [C.POINTER(LshConfig), f64p, f64p, u64p, u64p, C.c_char_p, C.c_size_t]),
    "genie_encoder_create": (C.c_int, [C.POINTER(LshConfig), C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "genie_encoder_destroy": (None, [vp]),
    "genie_lsh_encode": (C.c_int, [vp, f32p, C.c_uint64, u32p, C.c_char_p, C.c_size_t]),
    "genie_lsh_encode_device": (C.c_int, [vp, vp, C.c_uint64, vp, vp, C.c_char_p, C.c_size_t]),
    "genie_minhash_encode": (C.c_int, [vp, u64p, u64p, C.c_uint64, u32p, C.c_char_p, C.c_size_t]),
    "genie_minhash_encode_device": (C.c_int, [vp, vp, vp, C.c_uint64, vp, vp, C.c_char_p, C.c_size_t]),
    "genie_index_from_tokens_device": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                                 C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "genie_index_export": (C.c_int, [vp, u64p, u64p, u32p, C.c_char_p, C.c_size_t]),
    "genie_lsh_query_batch": (C.c_int, [vp, vp, C.POINTER(Config), vp, vp, vp, C.c_uint64, C.c_uint32,
                                        C.c_uint32, C.c_uint32, vp, vp, vp, C.POINTER(BatchStats),
                                        C.c_char_p, C.c_size_t]),
    "genie_mcix_parse_spans": (C.c_int, [vp, C.c_uint64, u64p, u16p, u64p, C.c_char_p, C.c_size_t]),
    "genie_mcix_serialize_spans": (C.c_int, [C.c_uint32, C.c_uint64, u64p, u16p, u64p, C.c_uint64, u32p, vp, u64p,
                                             C.c_char_p, C.c_size_t]),
    "genie_merge_topk_device_layout": (C.c_int, [vp, C.c_uint32, C.c_uint32, vp, vp, C.c_uint32, C.c_uint32, vp,
                                                 C.c_uint32, vp, vp, vp, vp, C.c_char_p, C.c_size_t]),
    "genie_group_create": (C.c_int, [C.c_uint32, C.c_uint64, u64p, u64p, u32p, C.c_uint32, C.POINTER(C.c_int),
                                     C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "genie_group_from_indexes": (C.c_int, [C.POINTER(vp), u32p, C.c_uint32, C.c_int, C.POINTER(vp), C.c_char_p,
                                           C.c_size_t]),
    "genie_group_destroy": (None, [vp]),
    "genie_group_info": (C.c_int, [vp, u32p, C.POINTER(C.c_int), u32p]),
    "genie_seqset_create": (C.c_int, [vp, u64p, C.c_uint64, C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "genie_seqset_destroy": (None, [vp]),
    "genie_seqset_info": (None, [vp, u64p, u64p, C.POINTER(C.c_int)]),
    "genie_seqset_distances": (C.c_int, [vp, vp, C.c_uint64, u32p, C.c_uint64, C.c_uint32, u32p, C.c_char_p,
                                         C.c_size_t]),
    "genie_group_query_batch": (C.c_int, [vp, C.POINTER(Config), C.c_uint32, u32p, u32p, u64p, u16p, u32p, u32p,
                                          C.c_uint32, C.POINTER(Entry), u32p, u32p, C.POINTER(StageNs),
                                          C.POINTER(BatchStats), C.c_char_p, C.c_size_t]),
}

GENIE_EXCHANGE_AUTO = 0
GENIE_EXCHANGE_NCCL = 1
GENIE_EXCHANGE_PEER = 2

SYNTH_SYMBOLS = {
    "genie_synth_adult": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(vp)]),
    "genie_synth_tweets": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                     C.POINTER(vp)]),
    "genie_synth_sift": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(vp)]),
    "genie_synth_ocr": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(vp)]),
    "genie_synth_sets": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(vp)]),
    "genie_synth_random": (C.c_int, [C.c_uint32] * 8 + [C.c_uint64, C.POINTER(vp)]),
    "genie_dataset_free": (None, [vp]),
    "genie_dataset_csr": (None, [vp, u32p, u64p, C.POINTER(u64p), C.POINTER(u64p), C.POINTER(u32p)]),
    "genie_dataset_queries": (None, [vp, u32p, C.POINTER(u32p), C.POINTER(u32p), C.POINTER(u64p),
                                     C.POINTER(u16p), C.POINTER(u32p), C.POINTER(u32p)]),
    "genie_dataset_points": (None, [vp, u32p, u32p, C.POINTER(f32p), u32p, C.POINTER(f32p), C.POINTER(u32p),
                                    C.POINTER(u32p)]),
    "genie_dataset_sets": (None, [vp, u32p, C.POINTER(u64p), C.POINTER(u64p), u32p, C.POINTER(u64p),
                                  C.POINTER(u64p)]),
    "genie_synth_csr_from_objects": (C.c_int, [C.c_uint32, u64p, u16p, u32p, C.POINTER(vp), C.c_char_p,
                                               C.c_size_t]),
}


def _load(path: Path, symbols: dict) -> C.CDLL:
    if not path.exists():
        raise ImportError(
            f"{path.name} is not built ({path}); run `python -c 'import __graft_entry__ as g; g.build()'` "
            "-- the engine has no CPU fallback"
        )
    lib = C.CDLL(str(path), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
    for name, (res, args) in symbols.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_engine = None
_synth = None


def engine() -> C.CDLL:
    global _engine
    if _engine is None:
        _engine = _load(ENGINE_LIB, ENGINE_SYMBOLS)
    return _engine


def synth() -> C.CDLL:
    global _synth
    if _synth is None:
        _synth = _load(SYNTH_LIB, SYNTH_SYMBOLS)
    return _synth
