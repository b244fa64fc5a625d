"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libmoespeq_ref.so (the reference's
unmodified control-plane core + oracle/ref_shim.cpp).  Build with `make -C oracle -j8`."""
import ctypes
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_ref", "libmoespeq_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(_LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {_LIB_PATH} (make -C oracle)")
        L = ctypes.CDLL(_LIB_PATH)
        c = ctypes.c_char_p
        v = ctypes.c_void_p
        L.ref_last_error.restype = c
        L.ref_free.argtypes = [v]
        L.ref_generate_trace.restype = v
        L.ref_generate_trace.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.c_int,
            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
            ctypes.c_ulonglong]
        L.ref_run_simulation.restype = v
        L.ref_run_simulation.argtypes = [c, c]
        L.ref_run_simulation_ex.restype = v
        L.ref_run_simulation_ex.argtypes = [c, c, ctypes.c_int]
        L.ref_plan_prefetch.restype = v
        L.ref_plan_prefetch.argtypes = [c, ctypes.c_int, c, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int]
        L.ref_select_victim.restype = v
        L.ref_select_victim.argtypes = [c, ctypes.c_int, c, ctypes.c_int, ctypes.c_int]
        L.ref_governor.restype = v
        L.ref_governor.argtypes = [c]
        L.ref_trace_analysis.restype = v
        L.ref_trace_analysis.argtypes = [c]
        L.ref_compare_policies.restype = v
        L.ref_compare_policies.argtypes = [c, c, c, c]
        L.ref_sweep_k.restype = v
        L.ref_sweep_k.argtypes = [c, c, c]
        _lib = L
    return _lib


class RefError(RuntimeError):
    pass


def _take(ptr) -> str:
    L = lib()
    if not ptr:
        raise RefError(L.ref_last_error().decode())
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    L.ref_free(ptr)
    return s


def generate_trace(L, N, top_k, tokens, hard=0.441, soft=0.468, mismatch=0.091, accept=0.8,
                   skew=1.0, seed=0, shared=0, expert_bytes=25_000_000) -> str:
    """generate_synthetic_trace (trace.cpp:319-399) -> reference JSONL text."""
    return _take(lib().ref_generate_trace(L, N, top_k, shared, expert_bytes, tokens, hard, soft,
                                          mismatch, accept, skew, seed))


def run_simulation(trace_jsonl: str, config: dict) -> dict:
    """run_simulation (sim.cpp:458-466) on a reference run-config dict -> SimReport JSON."""
    return json.loads(_take(lib().ref_run_simulation(trace_jsonl.encode(),
                                                     json.dumps(config).encode())))


def run_simulation_csv(trace_jsonl: str, config: dict) -> dict:
    return json.loads(_take(lib().ref_run_simulation_ex(trace_jsonl.encode(),
                                                        json.dumps(config).encode(), 1)))


def plan_prefetch(trace_jsonl: str, k: int, resident, budget=2, f1=0.25, f2=0.75, capacity=1 << 20):
    return json.loads(_take(lib().ref_plan_prefetch(trace_jsonl.encode(), k,
                                                    json.dumps(resident).encode(), budget, f1, f2,
                                                    capacity)))


def select_victim(trace_jsonl: str, k: int, resident, now: int, layer_filter: int = -1):
    return tuple(json.loads(_take(lib().ref_select_victim(trace_jsonl.encode(), k,
                                                          json.dumps(resident).encode(), now,
                                                          layer_filter))))


def governor(request: dict) -> dict:
    return json.loads(_take(lib().ref_governor(json.dumps(request).encode())))


def trace_analysis(trace_jsonl: str) -> dict:
    """classify_fidelity (both granularities) + layer_entropy per layer (trace.cpp:401-462)."""
    return json.loads(_take(lib().ref_trace_analysis(trace_jsonl.encode())))


def compare_policies(trace_jsonl: str, config: dict, policies, capacities) -> list:
    return json.loads(_take(lib().ref_compare_policies(trace_jsonl.encode(), json.dumps(config).encode(),
                                                       json.dumps(list(policies)).encode(),
                                                       json.dumps(list(capacities)).encode())))


def sweep_k(trace_jsonl: str, config: dict, ks) -> list:
    return json.loads(_take(lib().ref_sweep_k(trace_jsonl.encode(), json.dumps(config).encode(),
                                              json.dumps(list(ks)).encode())))
