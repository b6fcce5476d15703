"""CPU-side checks of the C ABI: the library loads without a GPU, exports
every symbol include/vmp.h declares, and NVRTC compiles generated robots."""

import ctypes
import re

import pytest

from paper_2309_14545_b200 import _native, codegen, load_robot, runtime


def header_functions():
    text = _native.INCLUDE.joinpath("vmp.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(vmp_[a-z_]+)\s*\(", text))


def test_library_loads_and_exports_header_symbols():
    L = _native.lib()
    declared = header_functions()
    assert declared == set(_native.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.vmp_version() >= 10000


def test_error_mapping_without_gpu():
    L = _native.lib()
    rc = L.vmp_validate(None, None, None, 0, 0, 0, None, None)
    assert rc == _native.VMP_EARG
    assert b"null" in L.vmp_last_error()
    with pytest.raises(ValueError):
        _native.check(rc)


def test_nvrtc_compiles_generated_robot(tmp_path):
    rob = load_robot("planar2")
    src = codegen.generate_source(rob.program, rob.pairs, "planar2")
    out = tmp_path / "planar2.cubin"
    rc = _native.lib().vmp_compile(src.encode(), b"planar2.cu", str(out).encode())
    assert rc == 0, _native.lib().vmp_last_error()
    assert out.read_bytes()[:4] == b"\x7fELF"


def test_nvrtc_reports_compile_errors(tmp_path):
    rc = _native.lib().vmp_compile(b"this is not cuda", b"bad.cu", str(tmp_path / "x").encode())
    assert rc == _native.VMP_ECOMPILE
    assert b"NVRTC" in _native.lib().vmp_last_error()


def test_generated_source_structure():
    rob = load_robot("arm7")
    src = codegen.generate_source(rob.program, rob.pairs)
    for k in ("vmp_fk_rows", "vmp_fk_spheres", "vmp_validate_p1_s1_g1", "vmp_motion_p0_s2_g1"):
        assert k in src
    lay = codegen.derive_layout(rob.program, rob.pairs)
    assert len(lay.fine) == 11 and len(lay.pairs) == 42 and len(lay.const_spheres) == 2
    # every listed sphere pair twice: group-culled (motion rake) and in expanded
    # form for the batch kernels (a packed test covers two partners of one sphere)
    assert src.count("ok &= vmp_clear_pair(") == 42
    assert 2 * src.count("ok &= vmp_clear_pair2(") + src.count("ok &= vmp_clear_pair_x(") == 42
    # bundled cubins were prebuilt by build()
    assert runtime.prepare(rob.program, rob.pairs).exists()


def test_algorithmic_flops_matches_survey():
    # config 1 = 151 + 11*32*8 + 42*8 = 3,303 flop / config
    rob = load_robot("arm7")
    f = codegen.algorithmic_flops(rob.program, rob.pairs, (32, 0, 0))
    assert f["fk"] == 151 and f["total"] == 3303


def test_motion_workspace_sizing():
    """Workspace = fixed part (header, queue words, 32,768 spare slots) + 136 bytes
    per edge (failure record, n, 8 slots); batches above 2^22 edges run in
    sub-batches on a 2^22-edge workspace (csrc/vmp.cu, csrc/vmp_abi.h)."""
    L = _native.lib()
    b = [int(L.vmp_motion_workspace_bytes(n)) for n in (0, 1, 4, 5, 4096, 1 << 22, 1 << 23)]
    fixed = b[0]
    assert fixed >= 16 * 32768 and fixed % 16 == 0
    assert b[1] == b[2] == fixed + 4 * 136 and b[3] == fixed + 8 * 136      # padded to 4 edges
    assert b[4] == fixed + 4096 * 136
    assert b[5] == b[6] == fixed + (1 << 22) * 136
    assert int(L.vmp_motion_workspace_bytes(-1)) == 0
