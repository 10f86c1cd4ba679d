"""The ctypes structs of _lib.py match the C ABI declared in
include/sgkkt_b200.h field by field (offsets and sizes from a gcc-compiled
probe of the header; CPU only) — a drifted field would silently pass wrong
pointers to the kernels."""

from __future__ import annotations

import ctypes
import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

PAIRS = {
    "sgk_pattern": "Pattern", "sgk_program": "Program", "sgk_view": "View", "sgk_pattern9": "Pattern9",
    "sgk_program9": "Program9", "sgk_trifactor": "TriFactor", "sgk_trigroups": "TriGroups",
    "sgk_segview": "SegView", "sgk_fastdiag": "FastDiag", "sgk_grid9": "Grid9", "sgk_triwide": "TriWide",
}


def _c_fields(text: str, name: str) -> list[str]:
    end = re.search(r"\}\s*" + name + r";", text).start()
    start = text.rfind("typedef struct {", 0, end) + len("typedef struct {")
    body = text[start:end]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        m = re.search(r"(\w+)\s*(\[\d+\])?$", decl)
        fields.append(m.group(1))
    return fields


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_ctypes_structs_match_header(tmp_path):
    from paper_2512_23804_b200 import _lib

    text = (ROOT / "include" / "sgkkt_b200.h").read_text()
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sgkkt_b200.h"', "int main(void) {"]
    for cname in PAIRS:
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in _c_fields(text, cname):
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        cname, field, val = line.split()
        got[(cname, field)] = int(val)
    for cname, pyname in PAIRS.items():
        cls = getattr(_lib, pyname)
        assert ctypes.sizeof(cls) == got[(cname, "size")], cname
        c_fields = _c_fields(text, cname)
        py_fields = [f[0] for f in cls._fields_]
        assert py_fields == c_fields, (cname, py_fields, c_fields)
        for f in c_fields:
            assert getattr(cls, f).offset == got[(cname, f)], (cname, f)
