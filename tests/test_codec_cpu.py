"""Host logic of the compact value codecs (blocks.value_codec_of): which
storage of a block's values is lossless (include/gridlp_b200.h
GRIDLP_VALS_*). No GPU needed."""

import numpy as np
import torch

from paper_2601_07628_b200 import native
from paper_2601_07628_b200.blocks import value_codec_of


def test_unit_values():
    assert value_codec_of(np.array([1.0, -1.0, 1.0])) == native.VALS_UNIT
    assert value_codec_of(np.zeros(0)) == native.VALS_UNIT          # empty: nothing to store


def test_float_exact_values():
    for v in ([1.0, 2.0, -3.0], [0.5, -0.25, 2.0 ** 100], [-0.0, 1.0], [np.inf, -np.inf, 1.0], [1.0, 0.0]):
        assert value_codec_of(np.array(v)) == native.VALS_F32, v


def test_values_needing_f64():
    for v in ([0.1, 1.0], [1.0, np.nan], [1.0, 1e-310], [1.0, 1e39], [1.0, 1.0 + 2.0 ** -30]):
        assert value_codec_of(np.array(v)) == native.VALS_F64, v


def test_chunked_scan_matches_one_pass(monkeypatch):
    """The scan runs in chunks (bounded temporaries on 2B-nnz blocks): a unit
    prefix followed by non-unit chunks must still be classified exactly."""
    import paper_2601_07628_b200.blocks as b

    monkeypatch.setattr(b, "_CODEC_CHUNK", 4)
    v = torch.tensor([1.0, -1.0, 1.0, 1.0, 1.0, -1.0, 3.0, 1.0, 1.0, 1.0], dtype=torch.float64)
    assert value_codec_of(v) == native.VALS_F32
    v[9] = 0.1
    assert value_codec_of(v) == native.VALS_F64
    v = torch.tensor([1.0] * 9 + [-1.0], dtype=torch.float64)
    assert value_codec_of(v) == native.VALS_UNIT


def test_struct_carries_codec_field():
    fields = [f for f, _ in native.Csr._fields_]
    assert fields[-2:] == ["val_codec", "launch_flags"]
    assert native.ABI_VERSION == 2
