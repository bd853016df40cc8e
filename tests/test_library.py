"""CPU-side checks of the boundary: librp.so loads, exports every symbol include/rp.h declares,
and (without a GPU) fails loudly instead of falling back to the CPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "rp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:rp_status|int32_t|const char \*|const rp_program \*)\s*(rp_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    import paper_1911_02373_b200 as rp
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(rp.lib(), n), n
    assert sorted(rp.EXPORTED) == names
    assert rp.abi_version() == 1


def test_struct_layouts_match_header():
    """ctypes mirrors of rp.h structs have the C sizes (x86-64 ABI)."""
    import ctypes as C
    import paper_1911_02373_b200 as rp
    assert C.sizeof(rp.rp_basis) == 4 * 3 + 4 + 8 * 2
    assert C.sizeof(rp.rp_xform) == 8 * 8 + 4 * 8
    assert C.sizeof(rp.rp_hw) == 4 * 4 + 8 * 2 + 8 * 8
    assert C.sizeof(rp.rp_fit_info) == 4 * 2 + 8 * 3 + 4 * 2


def test_no_cpu_fallback_without_gpu():
    import torch
    import paper_1911_02373_b200 as rp
    import synth
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert rp.device_count() == 0
    case = synth.tiny_sweep()
    with pytest.raises(rp.RPError) as ei:
        rp.eval_argmin(case.programs[0], case.D, case.F)
    assert ei.value.status == 2
    with pytest.raises(rp.RPError):
        rp.fit(np.ones((4, 1)), np.ones((1, 4)), [[0], [1]], [[0], [1]])


def test_invalid_arguments_rejected_before_launch():
    import paper_1911_02373_b200 as rp
    with pytest.raises(rp.RPError) as ei:
        rp.xform_from_box([2.0], [1.0])  # hi < lo
    assert ei.value.status == 1


def test_codegen_compiles_for_sm100a(tmp_path):
    """rp_codegen runs without a GPU (given the transform); its source is valid CUDA for sm_100a
    and carries the program's constants as exact hexadecimal immediates."""
    import copy
    import shutil
    import subprocess
    import oracle
    import paper_1911_02373_b200 as rp
    import synth
    spec = copy.deepcopy(synth.large_program())
    c, e = oracle.xform_from_box(spec.box_lo, spec.box_hi)
    spec.xform_c, spec.xform_e = list(c), list(e)
    src = rp.codegen(spec)
    assert float(spec.coef[0][1]).hex().replace("0x1.", "").rstrip("0")[:8] in src
    assert 'extern "C" __global__' in src and "rp_jit_argmin" in src
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("no nvcc")
    f = tmp_path / "gen.cu"
    f.write_text(src)
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-c", str(f), "-o", str(tmp_path / "gen.o")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_program_limits_rejected_without_gpu():
    """Host-side program checks (rp_codegen validates without a device): n_SM must fit the sweep's
    1/SM_act table (n_sm < 1024), and the MWP-CWP template needs 3 metrics."""
    import copy
    import oracle
    import paper_1911_02373_b200 as rp
    import synth
    spec = copy.deepcopy(synth.large_program())
    c, e = oracle.xform_from_box(spec.box_lo, spec.box_hi)
    spec.xform_c, spec.xform_e = list(c), list(e)
    rp.codegen(spec)  # valid as generated
    big = copy.deepcopy(spec)
    big.hw = dict(spec.hw, n_sm=1024)
    with pytest.raises(rp.RPError) as ei:
        rp.codegen(big)
    assert ei.value.status == 5  # RP_ERR_UNSUPPORTED
    ok = copy.deepcopy(spec)
    ok.hw = dict(spec.hw, n_sm=1023)
    rp.codegen(ok)


def test_program_save_load_roundtrip():
    """rp_program_save / rp_program_load (host only): exact round trip of every field, stable
    bytes, and loud failures on tampering, truncation and a foreign blob."""
    import copy
    import oracle  # (test infrastructure: the box transform, so no device call is needed)
    import paper_1911_02373_b200 as rp
    import synth
    for spec in (synth.large_program(), synth.polybench_sweep(nD=8).programs[2], synth.tiny_sweep().programs[0]):
        spec = copy.deepcopy(spec)
        c, e = oracle.xform_from_box(spec.box_lo, spec.box_hi)
        spec.xform_c, spec.xform_e = list(c), list(e)
        blob = rp.save_program(spec)
        back = rp.load_program(blob)
        ref = rp.Program(spec)
        assert (back.d, back.p, back.template) == (spec.d, spec.p, spec.template)
        for i in range(len(spec.coef)):
            assert np.array_equal(back.num_exp[i], np.asarray(spec.num_exp[i], dtype=np.int16))
            assert np.array_equal(back.den_exp[i], np.asarray(spec.den_exp[i], dtype=np.int16))
            assert np.asarray(spec.coef[i], dtype=np.float64).tobytes() == back.coef[i].tobytes()
        assert back.hw == {k: getattr(ref.c.hw, k) for k, _ in rp.rp_hw._fields_}
        assert (back.R, back.Z0, back.Z1) == (spec.R, spec.Z0, spec.Z1)
        assert list(back.xform_c) == list(ref.xform[0]) and list(back.xform_e) == list(ref.xform[1])
        assert rp.save_program(back) == blob  # the loaded program saves to the same bytes
        for bad in (blob[:-1], blob[:20], b"XX" + blob[2:], blob[:30] + bytes([blob[30] ^ 1]) + blob[31:]):
            with pytest.raises(rp.RPError):
                rp.load_program(bad)
