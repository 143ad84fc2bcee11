"""ctypes declarations for libbfsht_b200.so (include/bfsht_b200.h)."""
import ctypes

from . import pack

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64


def declare(lib):
    pack.declare(lib)
    lib.bfsht_last_error.restype = ctypes.c_char_p
    lib.bfsht_last_error.argtypes = []
    lib.bfsht_plan_upload.restype = _I
    lib.bfsht_plan_upload.argtypes = [_P, ctypes.POINTER(_P)]
    lib.bfsht_plan_wrap.restype = _I
    lib.bfsht_plan_wrap.argtypes = [ctypes.POINTER(_I64), ctypes.POINTER(_P),
                                    ctypes.POINTER(_P), ctypes.POINTER(_P)]
    lib.bfsht_plan_free.restype = None
    lib.bfsht_plan_free.argtypes = [_P]
    lib.bfsht_plan_arena.restype = _P
    lib.bfsht_plan_arena.argtypes = [_P]
    lib.bfsht_plan_launches.restype = _I64
    lib.bfsht_plan_launches.argtypes = [_P]
    lib.bfsht_alt_apply.restype = _I
    lib.bfsht_alt_apply.argtypes = [_P, _I, _P]
    lib.bfsht_alt_stage.restype = _I
    lib.bfsht_alt_stage.argtypes = [_P, _I, _I, _P]
    lib.bfsht_plan_chain_info.restype = _I
    lib.bfsht_plan_chain_info.argtypes = [_P, _I, _I, ctypes.POINTER(_I64)]
    lib.bfsht_alt_orders.restype = _I
    lib.bfsht_alt_orders.argtypes = [_P, _I, _P, _P, _P, _P]
    lib.bfsht_alt_fields.restype = _I
    lib.bfsht_alt_fields.argtypes = [_P, _I, _I, _P, _P, _P, _P, _P]
    lib.bfsht_alt_apply_wide.restype = _I
    lib.bfsht_alt_apply_wide.argtypes = [_P, _I, _P, _P]
    lib.bfsht_sht_batch.restype = _I
    lib.bfsht_sht_batch.argtypes = [_P, _I, _I, _P, _P, _P, _P, _P]
    lib.bfsht_half_apply.restype = _I
    lib.bfsht_half_apply.argtypes = [_P, _I, _I, _I, _P, _P, _P, _P]
    lib.bfsht_sht_forward.restype = _I
    lib.bfsht_sht_forward.argtypes = [_P, _P, _P, _P]
    lib.bfsht_sht_inverse.restype = _I
    lib.bfsht_sht_inverse.argtypes = [_P, _P, _P, _P, _P]
    lib.bfsht_dft_rows.restype = _I
    lib.bfsht_dft_rows.argtypes = [_I64, _I64, _I, _P, _P, _P]
    lib.bfsht_half_table_device.restype = _I
    lib.bfsht_half_table_device.argtypes = [_I, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P,
                                            ctypes.c_double, _P]
    lib.bfsht_reset_launches.restype = _I
    lib.bfsht_reset_launches.argtypes = [_P]
    for name in ("bfsht_shard_pack", "bfsht_shard_unpack"):
        getattr(lib, name).restype = _I
        getattr(lib, name).argtypes = [_P, _P, _P, _P]
    for name in ("bfsht_gather_entries", "bfsht_scatter_entries"):
        getattr(lib, name).restype = _I
        getattr(lib, name).argtypes = [_P, _P, _I64, _P, _P]
    lib.bfsht_synth_rows.restype = _I
    lib.bfsht_synth_rows.argtypes = [_P, _P, _P, _I64, _I64, _P, _P]
    lib.bfsht_anal_rows.restype = _I
    lib.bfsht_anal_rows.argtypes = [_P, _P, _P, _I64, _I64, _P, _P, _P]
    lib.bfsht_comm_unique_id.restype = _I
    lib.bfsht_comm_unique_id.argtypes = [_P]
    lib.bfsht_comm_init.restype = _I
    lib.bfsht_comm_init.argtypes = [_P, _I, _I, ctypes.POINTER(_P)]
    lib.bfsht_comm_free.restype = None
    lib.bfsht_comm_free.argtypes = [_P]
    lib.bfsht_alltoall_transpose.restype = _I
    lib.bfsht_alltoall_transpose.argtypes = [_P, _P, _P, _P, _P, _I64, _P]
    lib.bfsht_shard_orders.restype = _I
    lib.bfsht_shard_orders.argtypes = [_I, _I, _I, _P, _P]
    lib.bfsht_exchange_layout.restype = _I
    lib.bfsht_exchange_layout.argtypes = [_I, _I, _I, _P, _P, _P]
    lib.bfsht_sharded_create.restype = _I
    lib.bfsht_sharded_create.argtypes = [_P, _P, ctypes.POINTER(_P)]
    lib.bfsht_sharded_info.restype = _I64
    lib.bfsht_sharded_info.argtypes = [_P, _P]
    lib.bfsht_sharded_forward.restype = _I
    lib.bfsht_sharded_forward.argtypes = [_P, _P, _P, _P]
    lib.bfsht_sharded_inverse.restype = _I
    lib.bfsht_sharded_inverse.argtypes = [_P, _P, _P, _P, _P]
    lib.bfsht_sharded_free.restype = None
    lib.bfsht_sharded_free.argtypes = [_P]


# every symbol include/bfsht_b200.h declares (checked by tests on CPU)
EXPORTS = (
    "bfsht_pack_plan", "bfsht_packed_info", "bfsht_packed_arrays",
    "bfsht_packed_free", "bfsht_chain_schedule", "bfsht_chain_sched_arrays",
    "bfsht_chain_sched_free", "bfsht_host_last_error", "bfsht_rec_coeffs", "bfsht_regen_tile_host", "bfsht_last_error", "bfsht_plan_upload",
    "bfsht_plan_wrap", "bfsht_plan_free", "bfsht_plan_arena",
    "bfsht_alt_apply", "bfsht_alt_stage", "bfsht_plan_chain_info", "bfsht_alt_orders", "bfsht_alt_fields",
    "bfsht_half_apply", "bfsht_sht_batch", "bfsht_alt_apply_wide",
    "bfsht_sht_forward", "bfsht_sht_inverse", "bfsht_dft_rows", "bfsht_half_table_device",
    "bfsht_plan_launches",
    "bfsht_reset_launches", "bfsht_shard_pack", "bfsht_shard_unpack",
    "bfsht_gather_entries", "bfsht_scatter_entries", "bfsht_synth_rows",
    "bfsht_anal_rows", "bfsht_comm_unique_id", "bfsht_comm_init", "bfsht_comm_free",
    "bfsht_alltoall_transpose", "bfsht_shard_orders", "bfsht_exchange_layout",
    "bfsht_sharded_create", "bfsht_sharded_info", "bfsht_sharded_forward",
    "bfsht_sharded_inverse", "bfsht_sharded_free",
)


def check(lib, rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed ({rc}): "
                           f"{lib.bfsht_last_error().decode()}")
