"""ctypes binding of the in-tree CUDA library (include/rnnb.h).

There is no CPU fallback: if ``librnnb.so`` is missing or CUDA is not
available, every product entry point raises.  Build it with
``python -m paper_1803_11389_b200.build`` (``__graft_entry__.build()``).
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RNNB_LIB", os.path.join(HERE, "librnnb.so"))  # override for A/B timing only

OK, EINVAL, ECUDA, ENOMEM, EUNSUPPORTED, EFORMAT = 0, 1, 2, 3, 4, 5
SRU, QRNN = 1, 2
MODES = {"f32": 0, "f64": 1, "bf16": 2, "tf32": 3, "f32x3": 4}
DT_F32, DT_F64, DT_U64 = 0, 1, 2

# every symbol include/rnnb.h declares (checked by tests/test_abi.py)
SYMBOLS = (
    "rnnb_last_error", "rnnb_version", "rnnb_plan_blocks", "rnnb_stack_create",
    "rnnb_stack_destroy", "rnnb_stack_set_layer", "rnnb_forward", "rnnb_forward_host",
    "rnnb_gates", "rnnb_sweep", "rnnb_finalize", "rnnb_query", "rnnb_stack_create_ex",
    "rnnb_stack_set_highway", "rnnb_lstm_create", "rnnb_lstm_destroy", "rnnb_lstm_set_weights",
    "rnnb_lstm_forward", "rnnb_lstm_forward_host", "rnnb_lstm_query", "rnnb_rnnw_info",
    "rnnb_stack_load_rnnw", "rnnb_lstm_load_rnnw", "rnnb_rnnx_info", "rnnb_rnnx_load",
    "rnnb_forward_ex", "rnnb_dev_alloc", "rnnb_dev_free", "rnnb_ipc_handle", "rnnb_ipc_open",
    "rnnb_ipc_close", "rnnb_peer_access", "rnnb_flag_signal", "rnnb_flag_wait",
    "rnnb_gemm", "rnnb_activation", "rnnb_splitmix_uniform",
    "rnnb_linear_create", "rnnb_linear_destroy", "rnnb_linear_set_weights", "rnnb_linear_forward",
    "rnnb_linear_query", "rnnb_rnnw_read",
)
MAX_PEERS = 7
IPC_HANDLE_BYTES = 64
FLAG_WIDE_SRU = 1

_lib = None


class RnnbError(RuntimeError):
    pass


def load():
    """Load librnnb.so (once).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RnnbError(f"{LIB_PATH} is not built; run `python -m paper_1803_11389_b200.build` "
                        "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    P64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "rnnb_last_error": ([], ctypes.c_char_p),
        "rnnb_version": ([], ctypes.c_char_p),
        "rnnb_plan_blocks": ([i64, i64, P64, P64], ci),
        "rnnb_stack_create": ([ctypes.POINTER(vp), ci, ci, P64, P64, ci, ci], ci),
        "rnnb_stack_destroy": ([vp], ci),
        "rnnb_stack_create_ex": ([ctypes.POINTER(vp), ci, ci, P64, P64, ci, ci, ci], ci),
        "rnnb_stack_set_highway": ([vp, ci, i64], ci),
        "rnnb_stack_set_layer": ([vp, ci, ctypes.POINTER(vp), ci, ci], ci),
        "rnnb_forward": ([vp, vp, i64, i64, i64, vp, i64, vp, vp, vp], ci),
        "rnnb_forward_host": ([vp, vp, i64, i64, vp, vp, vp, vp], ci),
        "rnnb_gates": ([vp, ci, vp, i64, i64, vp, vp, i64, vp], ci),
        "rnnb_sweep": ([vp, vp, vp, vp, i64, i64, ci, vp], ci),
        "rnnb_finalize": ([ci, vp, vp, vp, vp, i64, i64, ci, vp], ci),
        "rnnb_query": ([vp, ci, ci, P64], ci),
        "rnnb_lstm_create": ([ctypes.POINTER(vp), i64, i64, ci, ci], ci),
        "rnnb_lstm_destroy": ([vp], ci),
        "rnnb_lstm_set_weights": ([vp, ctypes.POINTER(vp), ci, ci], ci),
        "rnnb_lstm_forward": ([vp, vp, i64, i64, i64, vp, i64, vp, vp, vp], ci),
        "rnnb_lstm_forward_host": ([vp, vp, i64, i64, vp, vp, vp, vp], ci),
        "rnnb_lstm_query": ([vp, ci, P64], ci),
        "rnnb_rnnw_info": ([ctypes.c_char_p, ctypes.POINTER(ci), ctypes.POINTER(ci), ctypes.POINTER(ci), P64, P64,
                            ci], ci),
        "rnnb_stack_load_rnnw": ([ctypes.POINTER(vp), ctypes.c_char_p, ci, ci], ci),
        "rnnb_lstm_load_rnnw": ([ctypes.POINTER(vp), ctypes.c_char_p, ci, ci, ci], ci),
        "rnnb_rnnx_info": ([ctypes.c_char_p, ctypes.POINTER(ci), P64, P64], ci),
        "rnnb_rnnx_load": ([ctypes.c_char_p, vp, ci, ci, vp], ci),
        "rnnb_forward_ex": ([vp, vp, i64, i64, i64, vp, i64, vp, vp, ci, ctypes.POINTER(vp), vp], ci),
        "rnnb_dev_alloc": ([ci, ctypes.c_size_t, ctypes.POINTER(vp)], ci),
        "rnnb_dev_free": ([ci, vp], ci),
        "rnnb_ipc_handle": ([vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64)], ci),
        "rnnb_ipc_open": ([ci, ctypes.c_char_p, ctypes.POINTER(vp)], ci),
        "rnnb_ipc_close": ([ci, vp], ci),
        "rnnb_peer_access": ([ci, ci], ci),
        "rnnb_flag_signal": ([ci, vp, ctypes.c_uint32, vp], ci),
        "rnnb_flag_wait": ([ci, vp, ctypes.c_uint32, vp], ci),
        "rnnb_gemm": ([ci, vp, i64, vp, i64, vp, i64, i64, i64, i64, ci, vp], ci),
        "rnnb_activation": ([ci, vp, vp, i64, ci, vp], ci),
        "rnnb_splitmix_uniform": ([ctypes.c_uint64, ctypes.c_uint64, i64, vp, ci, vp], ci),
        "rnnb_linear_create": ([ctypes.POINTER(vp), i64, i64, ci, ci], ci),
        "rnnb_linear_destroy": ([vp], ci),
        "rnnb_linear_set_weights": ([vp, vp, vp, ci], ci),
        "rnnb_linear_forward": ([vp, vp, i64, i64, vp, i64, vp], ci),
        "rnnb_linear_query": ([vp, ci, P64], ci),
        "rnnb_rnnw_read": ([ctypes.c_char_p, vp, i64, ci], ci),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def check(status):
    """Map a status code to the reference's exception types."""
    if status == OK:
        return
    msg = load().rnnb_last_error().decode(errors="replace")
    if status == EFORMAT:
        from . import model_io
        cls, _, text = msg.partition(": ")
        raise getattr(model_io, cls, model_io.FileFormatError)(text or msg)
    if status == EINVAL:
        raise ValueError(msg)
    raise RnnbError(f"rnnb status {status}: {msg}")
