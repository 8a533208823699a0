"""The tensor-core (sparse FP4 tcgen05) ID-level encoder prototype
(csrc/hv_encode_tc.cu, opt-in with HVB200_ENCODE_TC=1) against the table
encoder, which the reference goldens pin: odd and even feature counts (the
tiebreak), partial M tiles, D not a multiple of the N tile, both N widths
(192 and 128), pitched rows and row padding bytes that are not bins."""
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

dv = pytest.importorskip("paper_2206_04746_b200.device")


def _encode(eng, b8, tc, n128=False):
    old = {k: os.environ.get(k) for k in ("HVB200_ENCODE_TC", "HVB200_TC_N")}
    try:
        os.environ.pop("HVB200_ENCODE_TC", None)
        os.environ.pop("HVB200_TC_N", None)
        if tc:
            os.environ["HVB200_ENCODE_TC"] = "1"
        if n128:
            os.environ["HVB200_TC_N"] = "128"
        return eng.encode(b8, pitched=True)
    finally:
        for k, v in old.items():
            os.environ.pop(k, None)
            if v is not None:
                os.environ[k] = v


@pytest.mark.parametrize("F,D,rows", [(8, 256, 128), (342, 10000, 3000), (343, 1000, 5000), (561, 10000, 700),
                                      (784, 20000, 300), (617, 32768, 260), (100, 130, 1000)])
def test_tc_encoder_matches_table_encoder(F, D, rows):
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=F * 7 + D)
    eng = dv.Engine(cbk, 2)
    b8, _ = eng.synth(0, rows, 0, 5)
    ref = _encode(eng, b8, False)
    assert torch.equal(_encode(eng, b8, True), ref)
    assert torch.equal(_encode(eng, b8, True, n128=True), ref)


def test_tc_encoder_ignores_row_padding_bytes():
    F, D, rows = 342, 2000, 1000
    cbk = dv.DeviceCodebook.make(F, 16, D, seed=3)
    eng = dv.Engine(cbk, 2)
    b8, _ = eng.synth(0, rows, 0, 5)
    ref = _encode(eng, b8, False)
    noisy = b8.clone()
    noisy[:, F:] = torch.randint(0, 256, (rows, noisy.shape[1] - F), dtype=torch.uint8, device=noisy.device)
    assert torch.equal(_encode(eng, noisy, True), ref)
