"""CPU checks of the boundary: libtgv.so builds for sm_100a, loads, exports
every function include/tgv.h declares, and rejects invalid arguments before
touching a device (no compute calls here)."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = sorted(glob.glob(os.path.join(ROOT, "include", "*.h")))


def declared_functions():
    names = set()
    for h in HEADERS:
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names |= set(re.findall(r"\b(tgv_[a-z_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ["tgv_create", "tgv_load_histograms", "tgv_iterate", "tgv_read_u", "tgv_energy", "tgv_destroy",
              "tgv_get_unique_id", "tgv_status_string", "tgv_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2107_14790_b200 import tgv
    out = subprocess.run(["nm", "-D", "--defined-only", tgv.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tgv_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    from paper_2107_14790_b200 import bricks
    assert set(tgv.EXPORTS) | set(bricks.EXPORTS) == set(declared_functions())


def test_library_is_sm100a():
    from paper_2107_14790_b200 import tgv
    out = subprocess.run(["cuobjdump", "--list-elf", tgv.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_null_safety():
    from paper_2107_14790_b200 import tgv
    assert tgv.lib.tgv_status_string(0) == b"TGV_OK"
    assert b"EINVAL" in tgv.lib.tgv_status_string(-1)
    tgv.lib.tgv_destroy(None)  # NULL-safe
    assert tgv.lib.tgv_iterate(None, 1) == tgv.TGV_EINVAL


C8 = [-0.875 + 0.25 * b for b in range(8)]


@pytest.mark.parametrize("kw,frag", [
    (dict(tau=0.5, sigma=0.25), "tau*sigma*16"),
    (dict(tau=0.0), "tau and sigma"),
    (dict(lam=-1.0), ">= 0"),
    (dict(centers=[0.5, 0.2]), "increasing"),
    (dict(centers=[-1.5, 0.0]), "outside"),
    (dict(centers=[0.0] * 17), "nbins"),
    (dict(shape=(0, 4, 4)), "extents"),
    (dict(z_begin=2, z_end=2), "slab"),
    (dict(nranks=2, rank=0), "uid"),
    (dict(z_begin=1), "whole grid"),
    (dict(shape=(2048, 2048, 600)), "2^31"),  # one field of the slab would need >= 2^31 elements
])
def test_create_rejects_invalid_arguments(kw, frag):
    from paper_2107_14790_b200 import tgv
    args = dict(shape=(4, 4, 4), z_begin=0, z_end=None, centers=C8, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25,
                sigma=0.25, rank=0, nranks=1, uid=None, device=0)
    args.update(kw)
    if args["z_end"] is None:
        args["z_end"] = args["shape"][2]
    with pytest.raises(tgv.TgvError) as ei:
        tgv.tgv_create(args["shape"], args["z_begin"], args["z_end"], args["centers"], args["lam"], args["alpha0"],
                       args["alpha1"], args["tau"], args["sigma"], args["rank"], args["nranks"], args["uid"],
                       args["device"])
    assert ei.value.status == tgv.TGV_EINVAL
    assert frag in str(ei.value)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2107_14790_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "tgv_oracle", "oracle_"):
                    assert bad not in txt, (f, bad)


@pytest.mark.parametrize("kw,frag", [
    (dict(edge=6), "brick edge"),
    (dict(coords=[(0, 0, 0), (0, 0, 0)]), "duplicate"),
    (dict(coords=[(-1, 0, 0)]), "outside"),
    (dict(tau=0.5), "tau*sigma*16"),
    (dict(centers=[0.5, 0.2]), "increasing"),
    (dict(edge=32, coords=[(i % 256, i // 256, 0) for i in range(65536)]), "2^31"),
    (dict(levels=[0, 8]), "level"),  # tgv_bricks_create_mixed: levels <= 7
    (dict(levels=[1, 1], coords=[(0, 0, 0), (0, 0, 0)]), "duplicate"),  # same level and coordinates
])
def test_bricks_create_rejects_invalid_arguments(kw, frag):
    """include/tgv_bricks.h: argument checks happen before any device work."""
    from paper_2107_14790_b200 import tgv
    from paper_2107_14790_b200.bricks import BrickSolver
    args = dict(edge=8, coords=[(0, 0, 0), (1, 0, 0)], tau=0.25, centers=None, levels=None)
    args.update(kw)
    with pytest.raises(tgv.TgvError) as ei:
        BrickSolver(args["edge"], args["coords"], centers=args["centers"], tau=args["tau"], levels=args["levels"])
    assert ei.value.status == tgv.TGV_EINVAL
    assert frag in str(ei.value)
