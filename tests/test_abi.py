"""The C ABI library loads and exports every symbol include/cf.h declares
(no compute calls: CPU only)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "cf.h")) as f:
        text = f.read()
    return set(re.findall(r"CF_API\s+[\w\s\*]*?\b(cf\w+)\s*\(", text))


def test_header_declarations_match_binding_table():
    from paper_2504_09014_b200 import _lib
    assert _declared() == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2504_09014_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing


def test_status_codes_match_reference_error_codes():
    from paper_2504_09014_b200 import _lib, errors
    lib = _lib.lib()
    for i, code in enumerate(errors.STATUS_CODES):
        assert lib.cfStatusCode(i).decode() == code
    # every reference error class (cf/errors.py:6-93) has a status
    ref_codes = {"E_GENERIC", "E_BAD_SIZE", "E_NO_SEM", "E_BAD_DELTA", "E_OOB", "E_DEADLOCK",
                 "E_PROXY_DOWN", "E_ZERO_FLAG", "E_WRONG_PROTOCOL", "E_BAD_ALIGN", "E_SYNTAX",
                 "E_VERSION", "E_REF", "E_SHAPE", "E_PROTOCOL", "E_RANK_MISMATCH", "E_TOPOLOGY",
                 "E_NO_ALGO", "E_BAD_TIME", "E_CONFIG"}
    assert ref_codes <= set(errors.STATUS_CODES)
    assert lib.cfVersion() == 1


def test_raise_status_maps_classes():
    import pytest
    from paper_2504_09014_b200 import errors
    for i, code in enumerate(errors.STATUS_CODES[1:], start=1):
        with pytest.raises(errors.CommforgeError) as ei:
            errors.raise_status(i, "x")
        assert ei.value.code == code


def test_kernels_are_sm100a_cubins():
    """libcf.so carries sm_100a SASS (no PTX-only / other-arch fallback)."""
    import subprocess
    from paper_2504_09014_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if line.strip())


def test_config_rejects_threads_beyond_launch_bounds():
    """Every collective kernel is compiled with __launch_bounds__(512): larger
    CTAs are rejected at init (E_CONFIG), before any device is touched."""
    from paper_2504_09014_b200 import _lib, errors
    lib = _lib.lib()
    for threads in (1024, 544, 48, 100):
        cfg = _lib.cfConfig(threads=threads)
        comm = ctypes.c_void_p()
        devs = (ctypes.c_int * 2)(0, 0)
        st = lib.cfCommInitAll(ctypes.byref(comm), 2, devs, ctypes.byref(cfg))
        assert errors.STATUS_CODES[st] == "E_CONFIG", threads


def test_algo_ids_and_ring_transport_flag_match_header():
    """cfAlgo values and CF_ALGO_RING_LINKS in include/cf.h equal the Python
    table; variant "ring" of the three ring algorithms sets the flag, ""
    leaves it clear (all-pairs transport, same order and padding), any other
    variant is rejected like the reference rejects unknown variants."""
    import re
    from paper_2504_09014_b200 import _lib
    from paper_2504_09014_b200.collectives import _algo_id
    from paper_2504_09014_b200.errors import NoAlgoError
    hdr = open(os.path.join(ROOT, "include", "cf.h")).read()
    vals = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"CF_ALGO_(\w+) = (-?\d+)", hdr)}
    for name, v in _lib.ALGOS.items():
        assert vals[name] == v, name
    flag = int(re.search(r"#define CF_ALGO_RING_LINKS (0x[0-9a-f]+)", hdr).group(1), 16)
    assert flag == _lib.CF_ALGO_RING_LINKS
    for kind, name in (("allreduce", "2pr"), ("reducescatter", "ring_rs"), ("allgather", "ring_ag")):
        assert _algo_id(kind, name, "") == _lib.ALGOS[name]
        assert _algo_id(kind, name, "ring") == _lib.ALGOS[name] | flag
        with pytest.raises(NoAlgoError):
            _algo_id(kind, name, "port")
    with pytest.raises(NoAlgoError):
        _algo_id("allreduce", "2pa", "ring")
