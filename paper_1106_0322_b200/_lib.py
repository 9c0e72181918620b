"""ctypes binding of libspa_b200.so (declarations: include/spa_b200.h).

The library is the ONLY compute path: if it is missing or fails to load the
package raises, there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspa_b200.so")


class SpaDesign(ctypes.Structure):
    """Mirror of `spa_design` (include/spa_b200.h)."""

    _fields_ = [
        ("n", c_int32),
        ("q", c_int32),
        ("coded", c_int32),
        ("n_words", c_int32),
        ("planes", c_void_p),
        ("xcols", c_void_p),
        ("xlev", c_void_p),
        ("sy", c_void_p),
        ("alpha", c_void_p),
        ("gamma", c_void_p),
        ("penalized", c_void_p),
        ("gemm_b", c_void_p),
        ("kp", c_int32),
        ("terms", c_int32),
        ("codes", c_void_p),
        ("sx", c_void_p),
    ]


# name -> (restype, argtypes); every symbol the header declares.
_SIGNATURES = {
    "spa_last_error": (c_char_p, []),
    "spa_version": (c_int, []),
    "spa_philox_blocks": (c_int, [c_uint64, c_uint64, c_uint64, c_int64, c_void_p, c_void_p]),
    "spa_loglik_workspace_bytes": (c_size_t, [c_int64, c_int32]),
    "spa_k1_operand_bytes": (c_size_t, [POINTER(SpaDesign), c_int64]),
    "spa_loglik_softplus": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_void_p, c_void_p, c_size_t, c_void_p]),
    "spa_pack_particles": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_double,
                                   c_double, c_void_p, c_void_p]),
    "spa_loglik_rows": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_size_t, c_void_p]),
    "spa_prior_rows": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_int32, c_double, c_double, c_double, c_int32,
                               c_void_p, c_void_p]),
    "spa_prior_reweight": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_int32, c_double, c_double, c_double,
                                   c_void_p, c_void_p, c_void_p]),
    "spa_lse_chunk_stats": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "spa_lse_combine": (c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "spa_logw_apply": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "spa_resample_workspace_bytes": (c_size_t, [c_int64]),
    "spa_systematic_ancestors": (c_int, [c_void_p, c_int64, c_double, c_int64, c_int64, c_void_p, c_void_p, c_size_t,
                                         c_void_p]),
    "spa_exact_cumsum": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "spa_ipc_export": (c_int, [c_void_p, c_void_p, POINTER(c_uint64)]),
    "spa_ipc_open": (c_int, [c_void_p, POINTER(c_void_p)]),
    "spa_ipc_close": (c_int, [c_void_p]),
    "spa_copy_async": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "spa_resample_sharded": (c_int, [c_void_p, c_void_p, c_int32, c_int64, c_double, c_int32, c_void_p, c_void_p,
                                     c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_size_t, c_void_p]),
    "spa_resample_commit": (c_int, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_double, c_int64, c_void_p]),
    "spa_gather_rows": (c_int, [c_void_p, c_int32, c_void_p, c_int32, c_int32, c_void_p, c_int64, c_int64, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p]),
    "spa_summary_pass": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_int32, POINTER(c_double), c_int32,
                                 POINTER(c_double), c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p]),
    "spa_summary_select": (c_int, [c_void_p, c_int32, c_int32, POINTER(c_double), c_int32, c_void_p, c_void_p,
                                   c_void_p, c_void_p]),
    "spa_summary_finish": (c_int, [c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p]),
    "spa_format_particle_rows": (c_int, [c_void_p, c_void_p, c_int64, c_int32, c_int64, c_void_p, c_size_t,
                                         POINTER(c_size_t), c_int32]),
    "spa_em_map": (c_int, [POINTER(SpaDesign), c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int32,
                           c_double, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "spa_prepare": (c_int, []),
    "spa_step_record": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_void_p]),
    "spa_reweight_finish": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_double,
                                    c_void_p, c_void_p]),
    "spa_reweight_finish_max_particles": (c_int, []),
    "spa_resample_gated": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_void_p, c_void_p, c_int32, c_int32,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                   c_void_p]),
    "spa_mwg_resident_chains": (c_int, [POINTER(SpaDesign), POINTER(c_int64)]),
    "spa_mwg_set_rounds": (c_int, [c_int32, c_int32]),
    "spa_mwg_set_tables": (c_int, [c_int32]),
    "spa_mwg_chain_slots": (c_int, [c_void_p, c_void_p, c_int64, c_int32, c_double, c_double, c_double, c_int32,
                                    c_int32, c_uint64, c_int32, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p]),
    "spa_mwg_move": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_int32, c_double, c_double, c_double, c_int32,
                             c_uint64, c_int32, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int32,
                             c_void_p]),
    "spa_rw_moments_workspace_bytes": (c_size_t, [c_int64, c_int32]),
    "spa_rw_moments": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_int32, c_void_p, c_void_p,
                                c_size_t, c_void_p]),
    "spa_rw_factor": (c_int, [c_void_p, c_int32, c_double, c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p]),
    "spa_rw_normals": (c_int, [c_int64, c_int32, c_uint64, c_int64, c_int64, c_int32, c_void_p, c_void_p]),
    "spa_rw_propose": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_int32, c_void_p, c_uint64, c_int64, c_int64,
                               c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_void_p,
                               c_void_p]),
    "spa_rw_increments": (c_int, [c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "spa_rw_pack": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_double,
                            c_double, c_void_p, c_void_p]),
    "spa_tc_gemm_f32": (c_int, [c_void_p, c_int64, c_int32, c_void_p, c_int32, c_int32, c_void_p, c_int32, c_void_p]),
    "spa_rw_accept": (c_int, [c_void_p, c_int32, c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_uint64, c_int64, c_int64, c_int32, c_void_p, c_void_p]),
    "spa_loglik_partials": (c_int, [POINTER(SpaDesign), c_void_p, c_int64, c_void_p, c_size_t, c_void_p]),
    "spa_rw_accept_k1": (c_int, [c_void_p, c_int32, c_void_p, c_int32, c_int64, POINTER(SpaDesign), c_void_p,
                                 c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_int64, c_int64,
                                 c_int32, c_void_p, c_void_p]),
}

_lib = None


class SpaLibraryError(RuntimeError):
    """A libspa_b200 entry point returned a non-zero status."""


def load(path: str = LIB_PATH):
    """Load (once) and return the configured CDLL.  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SPA_B200_LIB", path)  # developer override (A/B builds)
    if not os.path.exists(path):
        raise RuntimeError(
            f"libspa_b200.so not found at {path}: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return list(_SIGNATURES)


# kernels launched by one call of each entry point (for bench.py's
# `gpu_launches`; csrc/*.cu are the source of truth)
KERNELS_PER_CALL = {
    "spa_philox_blocks": 1, "spa_loglik_softplus": 2, "spa_pack_particles": 1, "spa_loglik_rows": 3,
    "spa_prior_rows": 1, "spa_prior_reweight": 1, "spa_lse_chunk_stats": 1, "spa_lse_combine": 1, "spa_logw_apply": 1,
    "spa_systematic_ancestors": 4, "spa_exact_cumsum": 3, "spa_gather_rows": 1, "spa_mwg_move": 1, "spa_mwg_chain_slots": 1, "spa_rw_moments": 1,
    "spa_rw_factor": 0, "spa_mwg_resident_chains": 0, "spa_mwg_set_rounds": 0, "spa_mwg_set_tables": 0, "spa_step_record": 1, "spa_reweight_finish": 1, "spa_reweight_finish_max_particles": 0, "spa_resample_gated": 6, "spa_resample_sharded": 5, "spa_resample_commit": 1, "spa_summary_pass": 1, "spa_summary_select": 1,
    "spa_summary_finish": 1, "spa_em_map": 1, "spa_rw_propose": 2, "spa_rw_increments": 1, "spa_rw_pack": 1, "spa_rw_normals": 1, "spa_rw_accept": 1, "spa_loglik_partials": 1, "spa_rw_accept_k1": 1, "spa_tc_gemm_f32": 1,
}
launch_count = 0


def add_launches(n: int) -> None:
    """Entry points whose launch count depends on the problem (spa_rw_factor,
    spa_rw_moments phase 1) report it here."""
    global launch_count
    launch_count += int(n)


def call(name: str, *args) -> None:
    """Invoke an int-returning entry point and raise on a non-zero status."""
    global launch_count
    lib = load()
    launch_count += KERNELS_PER_CALL.get(name, 0)
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.spa_last_error().decode(errors="replace")
        raise SpaLibraryError(f"{name} failed with status {rc}: {msg}")
