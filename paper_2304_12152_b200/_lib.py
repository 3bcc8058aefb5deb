"""ctypes binding of csrc/libhtb200.so (the C-ABI declared in include/htb200.h).

There is no fallback: if the library is missing or a call fails, an exception
is raised.  Status codes map to the reference's exception types:
HT_E_INVALID -> ValueError, HT_E_NONFINITE -> FloatingPointError
(nn.py:147-148), anything else -> RuntimeError.
"""

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HTB200_LIB") or os.path.join(HERE, "csrc", "libhtb200.so")

HT_OK, HT_E_INVALID, HT_E_NONFINITE, HT_E_CUDA, HT_E_UNSUPPORTED = 0, 1, 2, 3, 4

_vp, _i, _i64, _d = C.c_void_p, C.c_int, C.c_int64, C.c_double
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)

# name -> argtypes (restype is always c_int status unless noted)
SIGNATURES = {
    "ht_version": [],
    "ht_device_supported": [_i, _ip],
    "ht_rng_seed": [C.c_uint64, _u64p],
    "ht_rng_uniforms": [_u64p, _i64, _vp],
    "ht_rng_gaussians": [_u64p, _i64, _vp],
    "ht_rng_gaussians_f32": [_u64p, _i64, _vp],
    "ht_rng_jump": [_u64p, C.c_uint64],
    "ht_rng_gaussians_device": [_u64p, _i64, _vp, _i, _vp],
    "ht_rng_uniforms_device": [_u64p, _i64, _vp, _i, _vp],
    "ht_rng_gaussian_maps_device": [_vp, _i, _i64, _vp, _i, _vp],
    "ht_num_params": [_i, _i, _i64p],
    "ht_packed_bytes": [_i, _i, _i64p],
    "ht_pack_params": [_vp, _i, _i, _vp, _vp],
    "ht_halftone_workspace_bytes": [_i, _i, _i, _i, _i, _i, _i, _i, _i64p],
    "ht_halftone": [_vp, _i, _i, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp,
                    _i64, _i, _vp],
    "ht_halftone_check": [_vp, _vp],
    "ht_multitone": [_vp, _i, _i, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i64,
                     _i, _vp],
    "ht_last_launch_count": [_ip],
    "ht_timing_enable": [_i],
    "ht_timing_reserve": [_i],
    "ht_timing_read": [_vp, _vp, _i, _ip],
    "ht_set_train_conv_impl": [_i],
    "ht_set_train_bits": [_i],
    "ht_set_wgrad_parts": [_i],
    "ht_set_edge_conv_impl": [_i],
    "ht_set_conv_pair": [_i],
    "ht_wgrad3x3_32": [_vp, _vp, _i, _i, _i, _vp, _vp, _i, _i, _vp],
    "ht_conv3x3_32": [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp],
    "ht_train_act_bytes": [_i, _i, _i, _i, _i, _i64p],
    "ht_policy_forward_train": [_vp, _i, _i, _vp, _i, _i, _i, _vp, _vp, _vp],
    "ht_policy_forward_train_async": [_vp, _i, _i, _vp, _i, _i, _i, _vp, _vp, _vp, _vp],
    "ht_policy_backward": [_vp, _i, _i, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp],
    "ht_reward_workspace_bytes": [_i, _i, _i, _i64p],
    "ht_reward_le": [_vp, _vp, _vp, _i, _i, _i, _vp, _i, _vp, _i, _d, _d, _d, _d, _d, _vp, _vp,
                     _vp, _vp, _i64, _vp],
    "ht_reward_signal": [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _i, _vp, _i, _d, _d, _d, _d, _i, _i,
                         _d, _vp, _vp, _vp, _vp, _i64, _vp],
    "ht_reinforce_signal": [_vp, _vp, _i, _i64, _vp, _d, _d, _vp, _vp],
    "ht_spectral_workspace_bytes": [_i, _i, _i, _i, _i64p],
    "ht_anisotropy": [_vp, _i, _i, _i, _vp, _vp, _i, _d, _vp, _vp, _vp, _i64, _vp],
    "ht_rapsd": [_vp, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i64, _vp],
    "ht_anisotropy_f64": [_vp, _i, _i, _i, _vp, _vp, _i, _d, _vp, _vp, _vp, _i64, _vp],
    "ht_rapsd_f64": [_vp, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i64, _vp],
    "ht_periodogram_f64": [_vp, _i, _i, _i, _vp, _vp, _i64, _vp],
    "ht_rapsd_power_f64": [_vp, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i64, _vp],
    "ht_reward_context_f64": [_vp, _vp, _i, _i, _i, _vp, _i, _vp, _i, _d, _d, _d, _d, _vp, _vp,
                              _vp, _vp, _vp],
    "ht_reward_delta_f64": [_vp, _vp, _vp, _i, _i, _i, _vp, _i, _vp, _i, _d, _d, _d, _d, _vp, _vp,
                            _i64, _vp],
    "ht_conv3x3_f64": [_vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp],
    "ht_conv3x3_f64_backward": [_vp, _vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp],
    "ht_adam_step": [_vp, _vp, _vp, _vp, _i64, _i, _d, _d, _d, _d, _vp],
    "ht_bin_gap_sum": [_vp, _i64, _vp, _vp],
}

_lib = None
_lock = threading.Lock()


def load():
    """Load (once) and return the CUDA library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not found: build it with `python -m paper_2304_12152_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib.ht_last_error.argtypes = []
        lib.ht_last_error.restype = C.c_char_p
        _lib = lib
        return lib


def check(rc, what=""):
    if rc == HT_OK:
        return
    msg = load().ht_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == HT_E_INVALID:
        raise ValueError(msg)
    if rc == HT_E_NONFINITE:
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


def call(name, *args):
    check(getattr(load(), name)(*args), name)


def out_i64(name, *args):
    v = C.c_int64(0)
    check(getattr(load(), name)(*args, C.byref(v)), name)
    return int(v.value)


def launch_count():
    v = C.c_int(0)
    load().ht_last_launch_count(C.byref(v))
    return int(v.value)


def ptr(t):
    """Device (or host) pointer of a torch tensor / numpy array, or None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2304_12152_b200 compute needs a CUDA device (sm_100a); "
                           "there is no CPU path")
    load()
