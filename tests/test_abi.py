"""The C ABI: every function include/resihp_b200.h declares is exported by the
built library and bound by the Python package, and the ctypes mirrors of the
descriptor structs have the C compiler's sizes and field offsets.  CPU only
(no compute calls)."""

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2605_06374_b200 import _lib, search

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "resihp_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rh_[a-z0-9_]+)\s*\(", text)))


def test_header_functions_are_exported_and_bound():
    lib = _lib.load_library()
    names = declared_functions()
    assert len(names) >= 20
    bound = set(_lib.EXPORTED_SYMBOLS) | set(search.EXPORTED_SYMBOLS)
    for n in names:
        assert hasattr(lib, n), f"{n} declared but not exported"
        assert n in bound, f"{n} not bound in Python"
    assert lib.rh_abi_version() == 1


STRUCTS = {
    "rh_cost_model": _lib.CostModelC,
    "rh_pipe_shape": _lib.PipeShape,
    "rh_segments": _lib.Segments,
    "rh_trace": _lib.Trace,
    "rh_trace_packed": _lib.TracePacked,
    "rh_pass_out": _lib.PassOut,
    "rh_screen_params": _lib.ScreenParams,
    "rh_migration_desc": _lib.MigrationDesc,
    "rh_search_desc": search.SearchDesc,
    "rh_candidate": search.Candidate,
}


def test_struct_layouts_match_c(tmp_path):
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(){"]
    for cname, py in STRUCTS.items():
        src.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            src.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    src.append("return 0;}")
    (tmp_path / "sz.c").write_text("\n".join(src))
    exe = tmp_path / "sz"
    subprocess.run(["gcc", str(tmp_path / "sz.c"), "-o", str(exe)], check=True)
    out = dict(line.rsplit(" ", 1) for line in subprocess.check_output([str(exe)]).decode().split("\n") if line)
    for cname, py in STRUCTS.items():
        assert int(out[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(out[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"


def test_no_gpu_means_loud_failure(monkeypatch):
    """Without a device the product refuses to run (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(_lib.BackendUnavailable):
        _lib.context()
