"""CPU checks of the boundary and host logic (no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2304_06543_b200 import _abi
from paper_2304_06543_b200.instance import PenaltySpec, ProblemInstance, ServiceCenter, SolverOptions
from paper_2304_06543_b200.sharded import shard_rows

HEADER = os.path.join(ROOT, "include", "lbdd_b200.h")
LIB = os.path.join(ROOT, "paper_2304_06543_b200", "lib", "liblbdd_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lbdd_b200_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build with `make -C paper_2304_06543_b200/csrc`"
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a():
    data = open(LIB, "rb").read()
    assert b"sm_100a" in data


def test_product_does_not_reference_oracle():
    # the oracle is test infrastructure only
    pkg = os.path.join(ROOT, "paper_2304_06543_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in text and "lbdd_oracle" not in text, f


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors vs the C compiler's view of include/lbdd_b200.h."""
    import subprocess
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "lbdd_b200.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu", sizeof(lbdd_instance_desc),'
                   'sizeof(lbdd_solver_options), sizeof(lbdd_solve_report),'
                   'offsetof(lbdd_solve_report, device_ns), offsetof(lbdd_solve_report, row_scan_ns));'
                   'return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    sizes = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                            check=True).stdout.split()]
    assert sizes == [ctypes.sizeof(_abi.InstanceDesc), ctypes.sizeof(_abi.SolverOptionsC),
                     ctypes.sizeof(_abi.SolveReportC), _abi.SolveReportC.device_ns.offset,
                     _abi.SolveReportC.row_scan_ns.offset]


def test_penalty_semantics():  # core.hpp:60-95
    assert PenaltySpec.constant(7).at(3) == 7 and PenaltySpec.constant(7).total(3) == 21
    lin = PenaltySpec.linear(5, 2)
    assert [lin.at(j) for j in (1, 2, 3)] == [5, 7, 9] and lin.total(3) == 21
    tab = PenaltySpec.table([3, 4, 9])
    assert [tab.at(j) for j in (1, 2, 3, 4, 5)] == [3, 4, 9, 9, 9] and tab.total(5) == 34
    assert PenaltySpec.constant(1).total(0) == 0


def test_solver_options_marshalling():
    c, keep = SolverOptions(parallel=True, refine_to_fixpoint=True, strict_order=[2, 0, 1]).to_c()
    assert c.parallel == 1 and c.refine_to_fixpoint == 1 and c.strict_order_len == 3
    assert [c.strict_order[i] for i in range(3)] == [2, 0, 1]


def test_error_mapping():
    for code, cls in [(1, ValueError), (2, _abi.LbddLogicError), (3, OverflowError), (4, RuntimeError)]:
        with pytest.raises(cls):
            _abi.raise_for(code, "x")
    _abi.raise_for(0, "")


def test_instance_rejects_out_of_int32_costs():
    with pytest.raises(_abi.LbddInvalidArgument):
        ProblemInstance([ServiceCenter(0, 1, PenaltySpec.constant(1))],
                        np.array([[2**31]], dtype=np.int64))


@pytest.mark.parametrize("n,world", [(10, 1), (10, 3), (7, 8), (1_000_003, 8), (0, 2)])
def test_shard_rows_partition(n, world):
    spans = [shard_rows(n, world, r) for r in range(world)]
    assert sum(r for _, r in spans) == n
    pos = 0
    for row0, rows in spans:
        assert row0 == pos and rows >= 0
        pos += rows
    assert max(r for _, r in spans) - min(r for _, r in spans) <= 1


REF_INCLUDE = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF_INCLUDE, "lbdd")),
                    reason="reference headers only exist in the build container")
def test_compat_header_compiles_against_reference_types(tmp_path):
    """include/lbdd_b200_compat.hpp is a drop-in for lbdd::asral_solve & co:
    it must compile against the reference's own headers and link the C ABI."""
    import subprocess
    src = tmp_path / "use.cpp"
    src.write_text(
        '#include "lbdd_b200_compat.hpp"\n'
        "int main() {\n"
        "  lbdd::ProblemInstance inst;\n"
        "  lbdd::SolveReport (*a)(const lbdd::ProblemInstance&, const lbdd::SolverOptions&, int) =\n"
        "      &lbdd::b200::asral_solve;\n"
        "  (void)a; (void)&lbdd::b200::strict_solve; (void)&lbdd::b200::greedy_solve;\n"
        "  return inst.n() == 0 ? 0 : 1;\n}\n")
    lib = os.path.join(ROOT, "paper_2304_06543_b200", "lib")
    out = subprocess.run(["g++", "-std=c++20", "-I", REF_INCLUDE, "-I", os.path.join(ROOT, "include"),
                          str(src), "-L", lib, "-llbdd_b200", "-o", str(tmp_path / "use")],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
