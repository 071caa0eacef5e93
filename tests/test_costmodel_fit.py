"""f1 pinned: the B200-measured step profiles fitted by the product library's
isim_model_fit_csv give the same cost model, bit for bit, as the reference
library's (proj/src/cost_model.cpp:100-157 fit_profile / load_profile_csv,
proj/src/capi.cpp:176-192), and the committed fitted JSON is that result.

The profiles are what tools/fit_costmodel.py measured on a B200
(profiles/costmodel/<preset>_profile.csv); also checked on edge-case CSVs
(too few points, all points below / above the saturation search range, a
malformed row -> the same status code and message from both libraries).
"""
import ctypes
import json
import os

import pytest

from conftest import PRODUCT_LIB, REF_LIB, ROOT

pytestmark = pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")


def _fit(lib_path, csv, base):
    L = ctypes.CDLL(lib_path)
    L.isim_model_fit_csv.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    L.isim_model_to_json.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    L.isim_model_free.argtypes = [ctypes.c_void_p]
    L.isim_string_free.argtypes = [ctypes.c_void_p]
    L.isim_last_error.restype = ctypes.c_char_p
    m = ctypes.c_void_p()
    st = L.isim_model_fit_csv(csv.encode(), base.encode() if base is not None else None, ctypes.byref(m))
    if st != 0:
        return st, L.isim_last_error().decode()
    s = ctypes.c_void_p()
    assert L.isim_model_to_json(m, ctypes.byref(s)) == 0
    out = ctypes.cast(s, ctypes.c_char_p).value.decode()
    L.isim_string_free(s)
    L.isim_model_free(m)
    return st, out


@pytest.mark.parametrize("preset", ["gptj-6b", "vicuna-13b"])
def test_fit_of_b200_profile_matches_reference(preset):
    csv = os.path.join(ROOT, "profiles", "costmodel", f"{preset}_profile.csv")
    m = {"gptj-6b": 458752, "vicuna-13b": 819200}[preset]
    base = json.dumps({"mem_per_token": m, "gpu_kv_capacity": 150e9, "cpu_kv_capacity": 128e9,
                       "swap_per_token": m / 50e9})
    ref = _fit(REF_LIB, csv, base)
    ours = _fit(PRODUCT_LIB, csv, base)
    assert ref[0] == 0 and ours == ref
    committed = json.load(open(os.path.join(ROOT, "profiles", "costmodel", f"{preset}_fitted.json")))
    fitted = json.loads(ours[1])
    for k in ("t0", "slope_below", "slope_above", "saturation_point"):
        assert fitted[k] == committed[k], k


@pytest.mark.parametrize("body", [
    "batch_tokens,seconds\n1,0.001\n",                                    # too few points
    "batch_tokens,seconds\n1,0.001\n2,0.002\n3,0.003\n4,0.004\n5,0.005\n",  # perfectly linear
    "batch_tokens,seconds\n1,0.001\nx,0.002\n3,0.003\n",                  # malformed row
    "batch_tokens,seconds\n",                                              # empty
    "batch_tokens,seconds\n4096,0.1\n8192,0.3\n16384,0.9\n32768,2.0\n",    # all large B
])
def test_fit_edge_cases_match_reference(tmp_path, body):
    csv = str(tmp_path / "p.csv")
    with open(csv, "w") as f:
        f.write(body)
    assert _fit(PRODUCT_LIB, csv, None) == _fit(REF_LIB, csv, None)
