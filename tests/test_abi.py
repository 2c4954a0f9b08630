"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/bicount_b200.h declares, ctypes layouts match the header,
and the product path refuses to run without a device (no CPU fallback)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2403_07858_b200 import _abi, build
from paper_2403_07858_b200.engine import EngineConfig, merge_limbs, split_limbs

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "bicount_b200.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _abi.open_library()


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(bc_\w+)\s*\(", text, re.M)))


def test_exports_every_declared_symbol(lib):
    declared = header_functions()
    assert set(declared) == set(_abi.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version_and_device_probe(lib):
    assert lib.bc_abi_version() == _abi.ABI_VERSION == 3
    assert lib.bc_device_count() >= 0


def test_struct_layout_matches_header():
    # bc_config: 8 x int32, then ptr/int64 pairs x 4 -> 32 + 64 = 96 bytes
    assert C.sizeof(_abi.BcConfig) == 96
    # bc_report: 2 u64 + 4 i32 + 18 i64 + 5 f64 + 3 i64 = 16 + 16 + 144 + 40 + 24
    assert C.sizeof(_abi.BcReport) == 240
    # and the C compiler agrees with ctypes on every field offset
    import subprocess
    import tempfile

    fields = [("bc_config", f) for f, _ in _abi.BcConfig._fields_] + [
        ("bc_report", f) for f, _ in _abi.BcReport._fields_]
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"bicount_b200.h\"\nint main(void){\n"
    src += 'printf("%zu %zu\\n", sizeof(bc_config), sizeof(bc_report));\n'
    for st, f in fields:
        src += f'printf("%zu\\n", offsetof({st}, {f}));\n'
    src += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c_file, exe = os.path.join(d, "t.c"), os.path.join(d, "t")
        open(c_file, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), "-o", exe, c_file], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    assert [int(x) for x in out[:2]] == [C.sizeof(_abi.BcConfig), C.sizeof(_abi.BcReport)]
    want = [getattr(_abi.BcConfig, f).offset for _, f in fields[:len(_abi.BcConfig._fields_)]]
    want += [getattr(_abi.BcReport, f).offset for _, f in fields[len(_abi.BcConfig._fields_):]]
    assert [int(x) for x in out[2:]] == want
    text = open(HEADER).read()
    cfg_body = re.search(r"typedef struct bc_config \{(.*?)\} bc_config;", text, re.S).group(1)
    names = re.findall(r"\*?(\w+)\s*(?:,|;)", re.sub(r"/\*.*?\*/", "", cfg_body, flags=re.S))
    assert [f for f, _ in _abi.BcConfig._fields_] == names
    rep_body = re.search(r"typedef struct bc_report \{(.*?)\} bc_report;", text, re.S).group(1)
    rep_names = re.findall(r"(\w+)\s*(?:,|;)", re.sub(r"/\*.*?\*/", "", rep_body, flags=re.S))
    assert [f for f, _ in _abi.BcReport._fields_] == rep_names


@pytest.mark.skipif(_abi.open_library().bc_device_count() > 0 if os.path.exists(_abi.LIB_PATH) else False,
                    reason="a GPU is present")
def test_no_cpu_fallback_without_device(lib):
    from paper_2403_07858_b200 import count_bicliques, synth

    with pytest.raises(RuntimeError, match="no CUDA device"):
        count_bicliques(synth.recon_graph(), 3, 2)


def test_invalid_arguments_fail_before_device(lib):
    from paper_2403_07858_b200 import count_bicliques, synth

    g = synth.recon_graph()
    with pytest.raises(ValueError):
        count_bicliques(g, 3, 2, EngineConfig(worker_count=0))
    with pytest.raises(ValueError):
        count_bicliques(g, 3, 2, EngineConfig(mode="bfs"))
    with pytest.raises(ValueError):
        count_bicliques(g, 3, 2, EngineConfig(anchor="W"))
    with pytest.raises(ValueError):
        count_bicliques(g, 0, 2)
    with pytest.raises(ValueError):
        count_bicliques(g, 3, 2, EngineConfig(shard_mode="diagonal"))
    with pytest.raises(ValueError):
        count_bicliques(g, 3, 2, EngineConfig(order_mode="fastest"))


@pytest.mark.parametrize("x", [0, 1, 2**32 - 1, 2**32, 2**64 + 5, 2**128 - 1, 90068795717])
def test_limbs_roundtrip(x):
    assert merge_limbs(split_limbs(x)) == x
    # summing limbs of several partials then normalising equals the exact sum
    parts = [x, (x * 7 + 3) % 2**126, 12345]
    summed = [sum(col) for col in zip(*(split_limbs(v) for v in parts))]
    assert merge_limbs(summed) == sum(parts)


def test_graph_csr_matches_reference_shape():
    from paper_2403_07858_b200 import synth

    g = synth.recon_graph()
    assert [a.tolist() for a in g.u_adj] == synth.RECON_U_NEIGHBORS
    assert g.edge_count == 14
    t = synth.transpose(g) if hasattr(synth, "transpose") else None
    from paper_2403_07858_b200.graph import transpose

    t = transpose(g)
    assert t.u_count == 5 and t.v_count == 4
    assert np.array_equal(t.u_csr.idx, g.v_csr.idx)


def test_integration_snippet_struct_layouts():
    """The reference-side binding shown in INTEGRATION.md declares bc_config / bc_report
    with the same fields, types and sizes as the library's own binding (and so the
    header): a stale snippet would hand bc_count a short struct."""
    import ctypes as C
    import re

    from paper_2403_07858_b200 import _abi

    text = open(os.path.join(os.path.dirname(os.path.dirname(HEADER)), "INTEGRATION.md")).read()
    ns = {"C": C}
    for name in ("_Cfg", "_Rep"):
        m = re.search(rf"class {name}\(C\.Structure\):.*?\n\n", text, re.S)
        assert m, name
        exec(m.group(0), ns)
    for mine, theirs in ((ns["_Cfg"], _abi.BcConfig), (ns["_Rep"], _abi.BcReport)):
        assert [(n, t) for n, t in mine._fields_] == [(n, t) for n, t in theirs._fields_]
        assert C.sizeof(mine) == C.sizeof(theirs)
