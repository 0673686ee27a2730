"""The ctypes mirrors of the C-ABI structs (paper_2304_06200_b200/_native.py) match the header
(include/leangrape_b200.h) field by field: offsets and sizes from a C program compiled with gcc."""

import os
import shutil
import subprocess
import tempfile

import pytest

from paper_2304_06200_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STRUCTS = {"lg_matrix": _native.lg_matrix, "lg_cost_term": _native.lg_cost_term,
           "lg_problem_desc": _native.lg_problem_desc}


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_ctypes_structs_match_header():
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "leangrape_b200.h"', "int main(void) {"]
    for name, cls in STRUCTS.items():
        lines.append(f'printf("{name} size %zu\\n", sizeof({name}));')
        for field, _ in cls._fields_:
            lines.append(f'printf("{name}.{field} %zu\\n", offsetof({name}, {field}));')
    lines.append("return 0; }")
    with tempfile.TemporaryDirectory() as tmp:
        src, exe = os.path.join(tmp, "layout.c"), os.path.join(tmp, "layout")
        with open(src, "w") as fh:
            fh.write("\n".join(lines))
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for name, cls in STRUCTS.items():
        assert int(got[f"{name} size"]) == __import__("ctypes").sizeof(cls), name
        for field, _ in cls._fields_:
            assert int(got[f"{name}.{field}"]) == getattr(cls, field).offset, (name, field)
