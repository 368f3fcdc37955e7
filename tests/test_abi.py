"""CPU-only checks of the C ABI boundary (no compute calls): the library
loads, exports every symbol include/pic.h declares, the ctypes mirror of
pic_config matches the C layout, the pure sizing call validates configs,
and there is no CPU fallback."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pic.h")
LIB = os.path.join(ROOT, "paper_1608_01009_b200", "libpic.so")


@pytest.fixture(scope="module")
def built():
    subprocess.check_call(["make", "-s", "-C", ROOT], stdout=subprocess.DEVNULL)
    assert os.path.exists(LIB)
    return C.CDLL(LIB)


def declared(header):
    src = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*\*?\s*(pic_\w+)\s*\(", src, re.M)))


def test_every_declared_symbol_is_exported(built):
    names = declared(HEADER)
    assert len(names) >= 12
    for n in names:
        assert hasattr(built, n), n
    out = subprocess.check_output(["nm", "-D", "--defined-only", LIB]).decode()
    exported = set(re.findall(r" T (pic_\w+)", out))
    assert set(names) <= exported


def test_binding_lists_every_symbol():
    from paper_1608_01009_b200 import EXPORTS
    assert sorted(EXPORTS) == declared(HEADER)


def test_oracle_exports_its_header(oracle_mod):
    names = re.findall(r"^\s*(?:int|void|double|int64_t)\s+(oracle_\w+)\s*\(",
                       open(os.path.join(ROOT, "oracle", "pic_oracle.h")).read(), re.M)
    L = oracle_mod.lib()
    for n in names:
        assert hasattr(L, n), n


@pytest.mark.parametrize("cname, pyname", [("pic_config", "PicConfig"), ("pic_diag", "PicDiag")])
def test_struct_layout_matches_c(tmp_path, cname, pyname):
    from paper_1608_01009_b200 import pic
    T = getattr(pic, pyname)
    fields = [f for f, _ in T._fields_]
    prog = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"',
            "int main(void){", f'printf("%zu\\n", sizeof({cname}));']
    prog += [f'printf("%zu\\n", offsetof({cname}, {f}));' for f in fields]
    prog += ["return 0;}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-o", str(exe), str(src)])
    vals = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert vals[0] == C.sizeof(T)
    for f, off in zip(fields, vals[1:]):
        assert getattr(T, f).offset == off, f


def _cfg(**kw):
    from paper_1608_01009_b200 import make_config
    args = dict(nx=16, ny=16, nz=16, species=[(-1.0, 1.0, 1e-4)], dt=0.5 / 3 ** 0.5,
                capacity=[32768], supercell=4, sort_every=5)
    args.update(kw)
    return make_config(**args)


def test_workspace_size_is_pure_and_validates(built):
    from paper_1608_01009_b200 import lib
    L = lib()
    nb = C.c_size_t(0)
    assert L.pic_workspace_size(C.byref(_cfg()), C.byref(nb)) == 0
    # E/B (6) + 2 x J (3) padded fields + 2 x 56 B per particle at least
    assert nb.value >= (12 * 20 * 20 * 20 * 8) + 2 * 56 * 32768
    big = C.c_size_t(0)
    assert L.pic_workspace_size(C.byref(_cfg(capacity=[10 * 32768])), C.byref(big)) == 0
    assert big.value > nb.value
    for h in (0, 1, 2):
        assert L.pic_workspace_size(C.byref(_cfg(halo=h)), C.byref(big)) == 0
    bad = [
        _cfg(dt=0.6),                      # CFL: 1/sqrt(3) = 0.577
        _cfg(supercell=3),                 # does not divide 16
        _cfg(species=[(-1.0, 0.0, 1.0)]),  # zero mass
        _cfg(nx=0),
        _cfg(halo=3),                      # tile drift halo h in {1, 2}
        _cfg(halo=-1),
    ]
    for b in bad:
        assert L.pic_workspace_size(C.byref(b), C.byref(nb)) == -1


def test_no_cpu_fallback(built):
    """Without a GPU, pic_init refuses (PIC_ECUDA) instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1608_01009_b200 import lib
    L = lib()
    ctx = C.c_void_p()
    buf = C.create_string_buffer(1 << 16)
    rc = L.pic_init(C.byref(_cfg()), C.cast(buf, C.c_void_p), 1 << 16, C.byref(ctx))
    assert rc in (-7, -2)
    assert not ctx.value


def test_product_does_not_touch_oracle():
    pkg = os.path.join(ROOT, "paper_1608_01009_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "pic_oracle" not in txt and "liboracle" not in txt, f
