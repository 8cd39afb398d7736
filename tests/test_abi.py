"""C-ABI library checks that need no GPU: it loads, exports every symbol the
header declares, and its host-side validator agrees with the paper's fixtures."""
import json
import os
import re

import numpy as np

import paper_2504_09590_b200 as bkv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _declared():
    src = open(os.path.join(ROOT, "include", "bkv.h")).read()
    return re.findall(r"BKV_API\s+[\w\s\*]+?\b(bkv_\w+)\s*\(", src)


def test_header_declares_the_survey_entry_points():
    names = set(_declared())
    assert {"bkv_kv_append", "bkv_paged_decode_attention", "bkv_decode_workspace_size",
            "bkv_validate_layout_host", "bkv_status_string", "bkv_last_error", "bkv_version"} <= names


def test_library_loads_and_exports_every_declared_symbol():
    L = bkv.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert L.bkv_version() >= 100
    assert L.bkv_status_string(0) == b"BKV_OK"
    assert L.bkv_status_string(4) == b"BKV_ERR_LAYOUT"


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bkv.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_host_validator_p711_and_a3b8():
    fx = json.load(open(os.path.join(GOLD, "p711_layout.json")))
    reqs = fx["requests"]
    M = max(len(r["block_table"]) for r in reqs)
    bt = np.full((len(reqs), M), -1, np.int32)
    for i, r in enumerate(reqs):
        bt[i, :len(r["block_table"])] = r["block_table"]
    dirs = np.array([r["dir"] for r in reqs], np.uint8)
    lens = np.array([r["len"] for r in reqs], np.int32)
    ok, info = bkv.validate_layout_host(bt, dirs, lens, fx["num_blocks"], fx["block_size"])
    assert ok, info
    fx = json.load(open(os.path.join(GOLD, "a3_b8_collision.json")))
    for c in fx["cases"]:
        M = max(len(c["B_bt"]), len(c["a_bt"]))
        bt = np.full((2, M), -1, np.int32)
        bt[0, :len(c["B_bt"])] = c["B_bt"]
        bt[1, :len(c["a_bt"])] = c["a_bt"]
        ok, info = bkv.validate_layout_host(bt, np.array([0, 1], np.uint8),
                                            np.array([c["B_len"], c["a_len"]], np.int32),
                                            c["num_blocks"], c["bs"])
        if c["expect_code"] == 0:
            assert ok
        else:
            assert not ok and info[0] == 2 and info[1:] == c["expect_info"]


def test_host_validator_rejections():
    bs = 16
    ok, info = bkv.validate_layout_host(np.array([[0, 1], [1, -1]], np.int32),
                                        np.array([[0, 0], [0, 0]], np.uint8), np.array([20, 2], np.int32), 3, bs)
    assert not ok and info[0] == 3
    ok, info = bkv.validate_layout_host(np.array([[0, 5]], np.int32), np.array([0], np.uint8),
                                        np.array([20], np.int32), 3, bs)
    assert not ok and info[0] == 1
    ok, info = bkv.validate_layout_host(np.array([[0]], np.int32), np.array([0], np.uint8),
                                        np.array([0], np.int32), 3, bs)
    assert not ok and info[0] == 1
    ok, _ = bkv.validate_layout_host(np.array([[0]], np.int32), np.array([0], np.uint8),
                                     np.array([0], np.int32), 3, bs, require_nonempty=False)
    assert ok


def test_host_validator_agrees_with_generator_layouts():
    from synth import make_case
    for cfg in ("tiny", "tiny_gqa", "opt13b", "llama70b"):
        lay = make_case(cfg, 5).layout
        ok, info = bkv.validate_layout_host(lay.block_tables, lay.dirs, lay.lens, lay.num_blocks, lay.block_size)
        assert ok, (cfg, info)


def test_no_cpu_fallback_for_device_calls():
    import torch
    import pytest
    pool = bkv.KVPool(torch.zeros(2, 1, 16, 64, dtype=torch.bfloat16), torch.zeros(2, 1, 16, 64, dtype=torch.bfloat16))
    with pytest.raises(bkv.BkvError):
        bkv.paged_decode_attention(pool, torch.zeros(1, 1, dtype=torch.int32), torch.zeros(1, dtype=torch.uint8),
                                   torch.ones(1, dtype=torch.int32), torch.zeros(1, 1, 64, dtype=torch.bfloat16))
