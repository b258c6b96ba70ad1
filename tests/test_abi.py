"""The C-ABI library builds, loads and exports every symbol include/hj.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hj.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hj_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_symbols()
    for n in ["hj_solve", "hj_coarse_feedback", "hj_label_subdomains", "hj_solve_partitioned",
              "hj_partition_plan", "hj_assign_subdomains", "hj_solve_workspace_bytes"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1405_3521_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    from paper_1405_3521_b200 import hj
    assert set(hj.EXPORTS) == set(declared_symbols())
    assert "sm_100a" in hj.hj_version()


def test_struct_layouts_match_header(tmp_path):
    """sizeof / offsetof of the ctypes mirrors equal what a C compiler sees in hj.h."""
    from paper_1405_3521_b200 import hj
    checks = {
        "hj_grid": ["dim", "periodic", "n", "lo", "hi"],
        "hj_problem": ["dynamics", "n_controls", "controls", "A", "b", "dubins_v", "lam", "h",
                       "l0", "lr", "v_out"],
        "hj_fields": ["speed", "piece", "g"],
        "hj_report": ["iterations", "residual", "converged", "node_updates", "device_ms",
                      "launches", "evaluated_updates"],
        "hj_subdomain": ["lo", "hi", "n_nodes", "box_nodes", "work"],
    }
    cname = {"lam": "lambda"}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "hj.h"', "int main(void){"]
    for st, fields in checks.items():
        lines.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fields:
            lines.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {cname.get(f, f)}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for st, fields in checks.items():
        cls = getattr(hj, st)
        assert ctypes.sizeof(cls) == int(got[st]), st
        for f in fields:
            assert getattr(cls, f).offset == int(got[f"{st}.{f}"]), (st, f)


def test_host_only_entry_points():
    """hj_assign_subdomains and the error path need no device."""
    from paper_1405_3521_b200 import hj
    plan = (hj.hj_subdomain * 5)()
    for k, w in enumerate([5.0, 1.0, 4.0, 3.0, 2.0]):
        plan[k].work = w
    # LPT: 5->r0, 4->r1, 3->r1 (7), 2->r0 (7), 1->r0 (tie -> lowest rank)
    assert hj.hj_assign_subdomains(plan, 2) == [0, 0, 1, 1, 0]
    assert hj.hj_assign_subdomains(plan, 1) == [0] * 5
    with pytest.raises(hj.HJError):
        hj.hj_assign_subdomains(plan, 0)
    assert "n_ranks" in hj.lib().hj_last_error().decode()


def test_product_has_no_cpu_fallback_and_no_oracle_import():
    """The product package never imports oracle/ and raises without the library."""
    pkg = os.path.join(ROOT, "paper_1405_3521_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn


def test_sweep_kernel_enum_matches_binding():
    """hj.h HJ_SWEEP_* values == the names hj.py marshals (sweep_kernel="...")."""
    from paper_1405_3521_b200 import hj
    src = open(os.path.join(ROOT, "include", "hj.h")).read()
    vals = {m.group(1).lower(): int(m.group(2))
            for m in re.finditer(r"HJ_SWEEP_([A-Z0-9_]+)\s*=\s*(\d+)", src)}
    assert vals == hj.SWEEP_KERNELS
