"""The C ABI boundary, checked without a GPU: the CUDA library builds for sm_100a,
loads, exports every entry point declared in include/scmwu.h, its structs have
the layout the ctypes binding assumes, and it fails loudly (no CPU fallback)
when no B200 is present."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2405_09157_b200 import _native as nat

HEADER = os.path.join(ROOT, "include", "scmwu.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sc_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def cuda_lib_path():
    path = os.path.join(nat.PKG_DIR, nat.LIB_NAME)
    if not os.path.exists(path):
        import build
        build.build_cuda()
    return path


def test_header_matches_binding():
    assert _declared() == sorted(nat.EXPORTS)


def test_cuda_library_exports_every_symbol(cuda_lib_path):
    lib = ctypes.CDLL(cuda_lib_path)
    for sym in _declared():
        assert hasattr(lib, sym), sym
    out = subprocess.run(["cuobjdump", "--list-elf", cuda_lib_path], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout, out.stdout[:500]


def test_checked_library_exports_every_symbol(cuda_lib_path):
    """libscmwu_checked.so (-DSCMWU_CHECKED, tests/test_gpu_checked.py) is the same ABI."""
    import build
    path = build.CHECKED_LIB
    if not os.path.exists(path):
        build.build_cuda(checked=True)
    lib = ctypes.CDLL(path)
    for sym in _declared():
        assert hasattr(lib, sym), sym
    # the checks are compiled into the checked library and out of the product library
    with open(path, "rb") as fh:
        assert b"SC_DCHECK failed" in fh.read()
    with open(cuda_lib_path, "rb") as fh:
        assert b"SC_DCHECK failed" not in fh.read()


def test_emulator_exports_every_symbol(emu_engine):
    for sym in _declared():
        assert hasattr(emu_engine.lib, sym), sym


def test_struct_layout_matches_header(tmp_path):
    prog = tmp_path / "layout.cpp"
    fields = {"sc_problem": nat.ScProblem, "sc_ftp_args": nat.ScFtpArgs,
              "sc_ftp_result": nat.ScFtpResult}
    lines = ['#include <cstdio>', '#include <cstddef>', f'#include "{HEADER}"', "int main(){"]
    for cname, cls in fields.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    prog.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["g++", "-o", str(exe), str(prog)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True,
                                                   text=True).stdout.splitlines())
    for cname, cls in fields.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, fname


def test_no_cpu_fallback_without_gpu(cuda_lib_path):
    """On a machine without a CUDA device the product raises; it never computes."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2405_09157_b200 import ses
    inst = ses.SesInstance(np.random.default_rng(0).standard_normal((10, 3)), np.zeros(10))
    with pytest.raises(nat.NativeUnavailable):
        ses.solve_ses(inst, 0.1)


def test_missing_library_raises(tmp_path):
    with pytest.raises(nat.NativeUnavailable):
        nat.Engine(str(tmp_path / "libscmwu.so"))


def test_bad_arguments_rejected(emu_engine):
    from paper_2405_09157_b200 import ses
    inst = ses.SesInstance(np.random.default_rng(0).standard_normal((10, 3)), np.zeros(10))
    dev = ses.ses_device(inst, engine=emu_engine)
    args = nat.ScFtpArgs(mode=nat.SC_MODE_REFINE, has_progress=1, alpha=1.0, horizon=0,
                         ceil_ln_r=3, delta=1e-4, patience=10, enabled=1, gain_rel=1e-4,
                         lo=-np.inf, hi=np.inf, target=np.nan)
    with pytest.raises(nat.NativeError):
        dev.handle.ftp(args)
    dev.close()


def test_integration_doc_binding_matches_header():
    """The ctypes structs of the reference-side binding (integration/_b200.py, the module
    INTEGRATION.md §2 drops into symcone/) must have exactly the fields of the package
    binding (itself checked against the header)."""
    import re
    doc = open(os.path.join(ROOT, "integration", "_b200.py")).read()
    block = doc[doc.index("class Problem(ctypes.Structure)"):doc.index("def enabled")]
    for cls, ours in (("Problem", nat.ScProblem), ("Args", nat.ScFtpArgs),
                      ("Result", nat.ScFtpResult)):
        body = block[block.index(f"class {cls}("):]
        body = body[:body.index("]") + 1]
        names = re.findall(r'\("(\w+)", ctypes\.c_\w+\)', body)
        assert names == [f[0] for f in ours._fields_], cls
