"""Run the measurement probes of tools/probe.cu (FP64 FMA peak, dependency latencies)."""
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def load():
    lib = ctypes.CDLL(os.path.join(HERE, "libprobe.so"))
    lib.mhdp_probe_fp64_peak.restype = ctypes.c_double
    lib.mhdp_probe_fp64_peak.argtypes = [ctypes.c_int]
    lib.mhdp_probe_latencies.restype = ctypes.c_int
    lib.mhdp_probe_latencies.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    lib.mhdp_probe_pivot_div.restype = ctypes.c_int
    lib.mhdp_probe_pivot_div.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_void_p]
    return lib


def pivot_div(x, piv, device=0):
    """PivotDiv(piv[j])(x[i]) on the device (k2_common.cuh), shape (len(piv), len(x))."""
    import numpy as np
    x = np.ascontiguousarray(x, dtype=np.float64)
    piv = np.ascontiguousarray(piv, dtype=np.float64)
    out = np.empty((piv.size, x.size), dtype=np.float64)
    st = load().mhdp_probe_pivot_div(device, x.ctypes.data, x.size, piv.ctypes.data, piv.size, out.ctypes.data)
    if st:
        raise RuntimeError(f"probe failed ({st})")
    return out


def fp64_peak(device=0):
    return load().mhdp_probe_fp64_peak(device)


def latencies(device=0):
    out = (ctypes.c_double * 6)()
    st = load().mhdp_probe_latencies(device, out)
    if st:
        raise RuntimeError(f"probe failed ({st})")
    keys = ["dfma", "markstein_div", "shfl_plus_dfma", "ieee_div", "smem_roundtrip", "gmem_roundtrip"]
    return dict(zip(keys, list(out)))


if __name__ == "__main__":
    r = {"fp64_flops": fp64_peak(), "cycles": latencies()}
    print(json.dumps(r))
