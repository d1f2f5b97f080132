"""CPU checks of the drop-in boundary (no GPU needed, no compute calls):
libslapcu.so loads, exports every function include/slapcu.h declares, the
Python binding covers exactly that set, and the pure host entry points behave
like the reference's (names, error kinds)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "slapcu.h")
LIB = os.path.join(ROOT, "paper_2106_14402_b200", "libslapcu.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(slapcu_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        pytest.fail("libslapcu.so not built (python -m paper_2106_14402_b200._build)")
    from paper_2106_14402_b200 import _lib

    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    for s in declared():
        assert hasattr(lib, s)


def test_binding_covers_header():
    from paper_2106_14402_b200 import _lib

    assert sorted(_lib.symbol_names()) == declared()


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_status_names_match_reference_error_kinds(lib):
    # error.hpp:27-36 kinds
    names = {s: lib.slapcu_status_name(s).decode() for s in range(0, 11)}
    assert names[1] == "DimError" and names[2] == "ShapeError" and names[3] == "InternalError"
    assert names[4] == "NameError" and names[5] == "BudgetError" and names[6] == "IndexError"
    assert names[10] == "DeadlockError"


def test_semiring_and_alg_names(lib):
    out = C.c_int()
    assert lib.slapcu_semiring_from_name(b"plus_times", b"f64", C.byref(out)) == 0 and out.value == 0
    assert lib.slapcu_semiring_from_name(b"min_plus", b"i32", C.byref(out)) == 0 and out.value == 3
    assert lib.slapcu_semiring_from_name(b"or_and", b"u8", C.byref(out)) == 0 and out.value == 5
    assert lib.slapcu_semiring_from_name(b"nope", b"f64", C.byref(out)) == 4  # NameError
    # spgemm.hpp:19-24
    for i, n in enumerate((b"heap", b"hash", b"hybrid")):
        assert lib.slapcu_alg_from_name(n, C.byref(out)) == 0 and out.value == i
    assert lib.slapcu_alg_from_name(b"quick", C.byref(out)) == 4
    assert [lib.slapcu_semiring_value_size(s) for s in range(6)] == [8, 4, 8, 4, 8, 1]
    assert lib.slapcu_abi_version() == 1


def test_semiring_ids_shared_with_oracle():
    import oracle

    from paper_2106_14402_b200 import _lib

    assert (oracle.PLUS_TIMES_F64, oracle.PLUS_TIMES_F32, oracle.PLUS_TIMES_I64, oracle.MIN_PLUS_I32,
            oracle.MIN_PLUS_F64, oracle.OR_AND_U8) == (_lib.PLUS_TIMES_F64, _lib.PLUS_TIMES_F32, _lib.PLUS_TIMES_I64,
                                                        _lib.MIN_PLUS_I32, _lib.MIN_PLUS_F64, _lib.OR_AND_U8)


def test_null_arguments_are_rejected(lib):
    # no context -> InvalidArgument, never a crash
    assert lib.slapcu_estimate_flops(None, None, None, None, None) == 7
    assert lib.slapcu_ctx_create(None, 0, None) == 7


def test_python_mirror_names():
    import paper_2106_14402_b200 as P

    assert P.spgemm_alg_from_name("hash") == P.SpGemmAlg.hash
    with pytest.raises(P.errors.NameError_):
        P.spgemm_alg_from_name("bogus")
    assert P.semiring_from_name("min_plus", "i32") is P.MinPlusI32
