"""Host-side checks of the C ABI (no GPU): the library builds for sm_100a, loads, exports every symbol
include/fb.h declares, and the ctypes structs match the C layout."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2311_09265_b200 import build as B
from paper_2311_09265_b200 import fb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fb.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fb_\w+)\s*\(", text)))


def test_header_declares_the_boundary_calls():
    names = declared_functions()
    for required in ("fb_build_pyramid", "fb_nnf_estimate", "fb_remap", "fb_blend_window", "fb_interpolate_keyframes"):
        assert required in names
    assert sorted(fb.SYMBOLS) == names


def test_library_loads_and_exports_every_declared_symbol():
    lib = C.CDLL(B.build_library())
    for name in declared_functions():
        assert hasattr(lib, name), name
    # the binary is sm_100a code
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f'''#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(fb_match_cfg), offsetof(fb_match_cfg, alpha),
         offsetof(fb_match_cfg, seed), sizeof(fb_stats), sizeof(fb_pair_key), offsetof(fb_pair_key, task_tag));
  return 0; }}''')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-o", str(exe), str(src)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert vals == [C.sizeof(fb._Cfg), fb._Cfg.alpha.offset, fb._Cfg.seed.offset, C.sizeof(fb._Stats),
                    C.sizeof(fb._Key), fb._Key.task_tag.offset]


def test_pyramid_elems_pure_host():
    lib = fb.load_library()
    assert lib.fb_pyramid_elems(2, 8, 6, 2) == 4 * 2 * (48 + 12)
    assert lib.fb_pyramid_elems(1, 8, 6, 0) == 0


def test_null_context_is_rejected_without_a_gpu():
    lib = fb.load_library()
    assert lib.fb_set_workspace(None, None, 0) == 1
    assert lib.fb_launch_count(None) == 0
    assert lib.fb_last_error(None) == b"null context"


def test_context_creation_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        fb.Context(0)


def declared_param_counts():
    """{function: number of parameters} from include/fb.h prototypes."""
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    out = {}
    for name, params in re.findall(r"\b(fb_\w+)\s*\(([^;{]*?)\)\s*;", text, flags=re.S):
        params = params.strip()
        out[name] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_binding_argtypes_match_header_arity():
    """Every ctypes prototype of the binding passes exactly the parameters the header declares."""
    lib = fb.load_library()
    counts = declared_param_counts()
    assert set(counts) == set(fb.SYMBOLS)
    for name, n in counts.items():
        at = getattr(lib, name).argtypes
        assert at is not None and len(at) == n, (name, n, at and len(at))
