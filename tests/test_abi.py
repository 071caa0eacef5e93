"""The C ABI library loads and exports every symbol include/infercept_b200.h declares."""
import ctypes
import os
import re

from conftest import PRODUCT_LIB, ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "infercept_b200.h")).read()
    return sorted(set(re.findall(r"\b(isim_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(PRODUCT_LIB)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(header_symbols()) >= 24 + 15


def test_reference_symbols_are_a_subset():
    # Every entry point of the reference's interceptsim.h (24) is declared here.
    ref = ["isim_abi_version", "isim_status_name", "isim_last_error", "isim_string_free", "isim_trace_generate",
           "isim_trace_load", "isim_trace_save", "isim_trace_request_count", "isim_trace_stats_json",
           "isim_trace_free", "isim_model_default", "isim_model_from_json", "isim_model_load", "isim_model_fit_csv",
           "isim_model_to_json", "isim_model_save", "isim_model_t_fwd", "isim_model_t_swap", "isim_model_free",
           "isim_run", "isim_result_summary_json", "isim_result_write_requests_csv", "isim_result_metric",
           "isim_result_free"]
    assert set(ref) <= set(header_symbols())


def test_python_binding_matches_header():
    from paper_2402_01869_b200 import _abi
    assert sorted(_abi.EXPORTS) == header_symbols()


def test_abi_version_and_status_names():
    import paper_2402_01869_b200 as ib
    from paper_2402_01869_b200 import _abi
    assert ib.abi_version() == 1
    for code, name in _abi.STATUS_NAMES.items():
        assert _abi.lib.isim_status_name(code).decode() == name


def test_null_arguments_are_invalid_arg():
    from paper_2402_01869_b200 import _abi
    assert _abi.lib.isim_trace_generate(None, None) == 1
    assert _abi.lib.isim_last_error().decode() == "null argument"
    assert _abi.lib.isim_trace_request_count(None) == 0
    assert _abi.lib.isim_model_t_fwd(None, 3.0) == 0.0


def test_executor_without_gpu_fails_loudly():
    from conftest import have_gpu
    import paper_2402_01869_b200 as ib
    if have_gpu():
        return
    try:
        ib.Executor({"preset": "tiny"})
    except ib.IsimError as e:
        assert e.status == 10  # ISIM_ERR_DEVICE, never a silent CPU fallback
    else:
        raise AssertionError("executor created without a GPU")


def test_measured_clock_needs_the_executor_and_unknown_clock_is_config_error():
    # run_json "clock" (f2): "virtual" (default, reference parity), "device",
    # "wall".  A measured clock without the B200 executor is a config error,
    # never a silent fallback to the virtual clock.
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from conftest import C0_COST, C0_WORKLOAD
    import paper_2402_01869_b200 as ib
    t = ib.Trace.generate(dict(C0_WORKLOAD, request_count=4))
    m = ib.CostModel.from_json(C0_COST)
    a = ib.run(t, m, dict(policy="infercept")).summary()
    assert ib.run(t, m, dict(policy="infercept", clock="virtual")).summary() == a
    for bad, text in ((dict(clock="device"), "needs the b200 executor"), (dict(clock="wall"), "needs the b200"),
                      (dict(clock="sundial"), "unknown clock")):
        try:
            ib.run(t, m, bad)
        except ib.IsimError as e:
            assert e.status == 2 and text in str(e), (bad, e)
        else:
            raise AssertionError(f"{bad} accepted")


def test_reference_capi_suite_links_against_product():
    """Drop-in proof: the reference's own C-API suite (proj/tests/test_capi.cpp:30-136),
    compiled unchanged, linked against OUR library instead of libinterceptsim.so."""
    import shutil
    import subprocess
    import pytest
    if not os.path.isdir("/root/reference/proj/tests") and not os.path.exists(
            os.path.join(ROOT, "oracle", "_ref", "obj", "test_capi.o")):
        pytest.skip("reference sources absent and no prebuilt test_capi.o")
    if shutil.which("make") is None:
        pytest.skip("make absent")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "product-capi"], check=True,
                   capture_output=True)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "capi_tests_product")], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "4 | 4 passed | 0 failed" in out.stdout, out.stdout
