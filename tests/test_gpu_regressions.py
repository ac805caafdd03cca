"""Regressions for defects found in review, each checked
against the oracle through the C-ABI."""
import numpy as np
import pytest

import paper_2507_11941_b200 as bb

pytestmark = pytest.mark.gpu


def _device_encode(enc, table, data, off):
    torch = pytest.importorskip("torch")
    n = off.size - 1
    total = int(off[-1])
    d = torch.from_numpy(np.ascontiguousarray(data)).cuda() if total else torch.zeros(1, dtype=torch.uint8,
                                                                                        device="cuda")
    o = torch.from_numpy(off.astype(np.int64)).cuda()
    ids = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
    oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    enc.encode_device(table, d.data_ptr(), o.data_ptr(), n, total, ids.data_ptr(), oo.data_ptr(), sync=True)
    oo = oo.cpu().numpy().view(np.uint64)
    return ids[: int(oo[-1])].cpu().numpy().view(np.uint32), oo


@pytest.mark.parametrize("path", ["device", "host"])
def test_trailing_empty_row_at_tile_end_leaves_no_row_bit(gpt2, oracle_for, path):
    """A batch of exactly 512 bytes followed by an empty row: the empty row
    starts at `total`, a tile boundary. Its row-start bit used to be set past
    the last tile (never cleared), then cut a later, longer encode on the same
    ctx at byte 512."""
    enc = bb.Encoder(device=0)
    text = (b"hello world, the quick brown fox jumps over the lazy dog. " * 64)
    big = bb.pack_rows([text[:1000]] * 2048)  # grows the scratch first
    a = bb.pack_rows([text[:512], b""])
    row = text[:1024]
    assert row[505:517] == b"er the lazy "  # " lazy" spans byte 512
    b = bb.pack_rows([row])
    orc = oracle_for("gpt2")
    for data, off in (big, a, b, a, b):
        if path == "device":
            ids, oo = _device_encode(enc, gpt2, data, off)
        else:
            ids, oo, _ = enc.encode_packed(gpt2, data, off)
        wi, wo = orc.encode_packed(data, off)
        assert np.array_equal(oo, wo)
        assert np.array_equal(ids, wi)


def test_block_bpe_ids_outside_table_never_pair(gpt2, oracle_for):
    """block_bpe on ids the table never mentions: an id >= 2^16 used to alias
    the narrow pair key (id 65536 + 5 behaved like id 5)."""
    orc = oracle_for("gpt2")
    h, e = gpt2.byte_token(ord("h")), gpt2.byte_token(ord("e"))
    assert orc.rank_of(h, e) is not None
    cases = [
        [h + 65536, e],
        [h, e, h + 65536, e, h, e],
        [h, h + (1 << 20), e, 0xFFFFFFF0, e, h, e],
        [70000, 70001, h, e, 70000],
    ]
    enc = bb.Encoder(device=0)
    for toks in cases:
        assert enc.block_bpe(gpt2, toks) == orc.block_bpe(toks), toks


def test_nonzero_first_offset_rejected(gpt2):
    """offsets[0] != 0 is a UsageError on every path (it used to encode the
    bytes before offsets[0] on the single-launch device path)."""
    torch = pytest.importorskip("torch")
    data = np.frombuffer(b"hello world, hello again", np.uint8).copy()
    off = np.array([3, 11, 24], np.uint64)
    d = torch.from_numpy(data).cuda()
    o = torch.from_numpy(off.astype(np.int64)).cuda()
    out = torch.empty(24, dtype=torch.int32, device="cuda")
    oo = torch.empty(3, dtype=torch.int64, device="cuda")
    with pytest.raises(bb.UsageError, match="start at 0"):
        bb.Encoder(0).encode_device(gpt2, d.data_ptr(), o.data_ptr(), 2, 24, out.data_ptr(), oo.data_ptr(),
                                    sync=True)
