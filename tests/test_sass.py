"""SASS checks of the built library (CPU only: cuobjdump on the .so).

* No kernel issues a global load before griddepcontrol.wait (SASS ACQBULK):
  with programmatic dependent launch a kernel starts while its predecessor is
  still running, and a hoisted ld.global.nc reads the previous iteration's
  data (this happened in K1 and faulted).
* The tensor-core kernels really are tcgen05 / TMA kernels (UTCHMMA / UTMALDG
  / LDTM in SASS), and the CTA-pair GEMM uses the 2-CTA forms.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2402_01869_b200", "libinfercept_b200.so")

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="needs cuobjdump")


def functions():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, name, body = {}, None, []
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = body
            name, body = m.group(1), []
        elif name:
            body.append(line)
    if name:
        funcs[name] = body
    return funcs


def test_no_global_load_before_grid_dependency_wait():
    bad = []
    for name, body in functions().items():
        text = "\n".join(body)
        if "ACQBULK" not in text:
            continue
        before = text.split("ACQBULK", 1)[0]
        if re.search(r"\bLDG\b|\bLDG\.", before):
            bad.append(name)
    assert not bad, f"global loads hoisted above griddepcontrol.wait in: {bad}"


def test_tensor_core_kernels_use_tcgen05_and_tma():
    funcs = functions()

    def sass_of(fragment):
        return "\n".join("\n".join(b) for n, b in funcs.items() if fragment in n)

    for frag in ("tc_gemm_pair_kernel", "tc_splitk_kernel", "chunk_attn_tc_kernel"):
        s = sass_of(frag)
        assert s, frag
        assert "UTCHMMA" in s and "UTMALDG" in s and "LDTM" in s, frag
    pair = sass_of("tc_gemm_pair_kernel")
    assert "UTCHMMA.2CTA" in pair and "UTMALDG.2D.2CTA" in pair
