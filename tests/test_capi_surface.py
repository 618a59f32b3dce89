"""The C-ABI library loads on a CPU-only host and exports every function the
public headers declare (no compute calls: those need a GPU)."""
import re
import subprocess
from pathlib import Path

import pytest

from paper_2602_11686_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared(header: Path):
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mp_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", ["moeplan.h", "moeplan_fsep.h"])
def test_header_symbols_exported(product_lib, header):
    names = declared(ROOT / "include" / header)
    assert names, header
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.lib_path())], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (mp_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_ctypes_table_covers_headers(product_lib):
    names = declared(ROOT / "include" / "moeplan.h") + declared(ROOT / "include" / "moeplan_fsep.h")
    assert set(names) <= set(_lib.exported_symbols())
    assert _lib.missing_symbols() == []


def test_status_names_and_last_error(product_lib):
    lib = product_lib
    assert lib.mp_status_name(0) == b"ok"
    assert lib.mp_status_name(4) == b"infeasible"
    assert lib.mp_status_name(7) == b"device"
    import ctypes as C
    h = C.c_void_p()
    st = lib.mp_config_parse(None, C.byref(h))
    assert st == 1 and b"NULL" in lib.mp_last_error()
    st = lib.mp_config_parse(b'{"topology": {"n_nodes": 1}}', C.byref(h))
    assert st == 2 and b"devices_per_node" in lib.mp_last_error()


def test_oracle_gap_status_and_output(product_lib):
    """mp_oracle_gap_json follows the ABI conventions: a config without a topology is
    invalid_argument (status 1) with the reason in mp_last_error; a complete config yields
    the JSON report (exact optimum <= greedy cost)."""
    import ctypes as C
    import json
    lib = product_lib
    cfg = C.c_void_p()
    assert lib.mp_config_parse(b'{"model": {"n_experts": 2, "capacity": 1}}', C.byref(cfg)) == 0
    out = C.c_void_p()
    assert lib.mp_oracle_gap_json(cfg, b'{"R": [[1, 2]]}', C.byref(out)) == 1
    assert b"topology" in lib.mp_last_error()
    lib.mp_config_free(cfg)
    full = json.dumps({"topology": {"n_nodes": 1, "devices_per_node": 2, "b_intra": 9e11, "b_inter": 9e11},
                       "cost": {"v_comm": 8192, "v_comp": 3.5e8, "b_comp": 1.6e15},
                       "model": {"n_experts": 2, "capacity": 1}, "planner": {"seed": 1}})
    assert lib.mp_config_parse(full.encode(), C.byref(cfg)) == 0
    assert lib.mp_oracle_gap_json(cfg, b'{"R": [[4, 2], [1, 3]]}', C.byref(out)) == 0
    rep = json.loads(C.cast(out, C.c_char_p).value.decode())
    lib.mp_string_free(out)
    assert rep["exact_cost"] <= rep["greedy_cost"] and rep["gap"] >= 1.0 and rep["layouts_examined"] == 2
    lib.mp_config_free(cfg)


def test_layer_create_fails_loudly_without_gpu(product_lib):
    """On a CPU-only host the layer must refuse (MP_ERR_DEVICE), never fall back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import ctypes as C
    d = _lib.FsepDesc(8, 2, 256, 256, 128, 8, 1, 0, 0, 0, 0)
    h = C.c_void_p()
    st = product_lib.mp_fsep_layer_create(C.byref(d), 0, C.byref(h))
    assert st == 7, st
