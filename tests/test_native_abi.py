"""CPU-side checks of the C-ABI library: it loads without a GPU and exports every symbol include/gllm.h declares."""
import ctypes as C
import os
import re

import pytest

from paper_2504_14775_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "gllm.h")).read()
    return sorted(set(re.findall(r"GLLM_API\s+[\w\s\*]+?\b(gllm_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2504_14775_b200 import build
    build.build()
    return native.load()


def test_exports_match_header(lib):
    declared = _declared()
    assert len(declared) >= 15
    assert sorted(native.EXPORTS) == declared
    for name in declared:
        assert hasattr(lib, name), name


def test_host_only_entry_points(lib):
    assert lib.gllm_version() >= 1
    assert lib.gllm_attention_q_tile(32, 8) == 64     # 2 tiles x 128 rows / G=4
    assert lib.gllm_attention_q_tile(40, 8) == 50
    assert lib.gllm_attention_q_tile(64, 8) == 32
    assert lib.gllm_attention_q_tile(3, 2) == -1
    d = native.Dims(32, 4096, 32, 8, 128, 14336, 128256, 0, 1e-5, 16, 1000, 64, 64, 1024, 3072, 1024)
    assert lib.gllm_stage_workspace_bytes(C.byref(d)) > 3072 * 4096 * 2


def test_errors_are_reported_not_crashing(lib):
    # NULL stage: rejected on the host before any CUDA call
    rc = lib.gllm_stage_forward(None, None, None)
    assert rc == 1 and b"null" in lib.gllm_last_error()
    with pytest.raises(native.NativeError):
        native.call("gllm_stage_forward", None, None, None)


def test_pack_batch_layout():
    """Host packer: seq_info / work / deltas / prompts land where include/gllm.h says."""
    import numpy as np

    from paper_2504_14775_b200.engine import BatchMeta, SeqMeta
    from paper_2504_14775_b200.stage import pack_batch
    meta = BatchMeta.from_seqs(3, [SeqMeta(7, 2, 40, 1, True), SeqMeta(9, 5, 0, 70, False), SeqMeta(4, 1, 10, 5, True)],
                               np.array([[5, 0, 11], [5, 1, 12]], np.int32), [(9, 5)])
    pb = pack_batch(meta, 32, lambda rid: np.arange(3, dtype=np.int32) + 100)
    assert (pb.n_seqs, pb.n_tokens, pb.n_emit, pb.n_work, pb.n_prefill_work, pb.n_deltas, pb.n_prompts) == (3, 76, 2, 5, 4, 2, 1)
    d = pb.data
    assert d[:15].tolist() == [2, 40, 1, 0, 0, 5, 0, 70, 1, -1, 1, 10, 5, 71, 1]
    assert d[15:25].tolist() == [1, 0, 1, 32, 1, 64, 2, 0, 0, 0]   # prefill tiles first, then decodes
    assert d[25:31].tolist() == [5, 0, 11, 5, 1, 12]
    assert d[31:34].tolist() == [5, 3, 0] and d[34:].tolist() == [100, 101, 102]
    assert pb.emit_ids == [7, 4] and pb.emit_pos == [41, 15]


def test_pad_decode_batch_layout():
    """CUDA-graph padding: real decodes keep their entries, padding sequences decode the scratch row."""
    import numpy as np

    from paper_2504_14775_b200.engine import BatchMeta, SeqMeta
    from paper_2504_14775_b200.stage import pack_batch, pad_decode_batch
    meta = BatchMeta.from_seqs(8, [SeqMeta(7, 2, 40, 1, True), SeqMeta(4, 1, 31, 1, True)],
                               np.array([[1, 2, 33]], np.int32), [])
    pb = pack_batch(meta, 32, lambda rid: None)
    pp = pad_decode_batch(pb, 4, scratch_row=50, scratch_page=900)
    assert (pp.n_seqs, pp.n_tokens, pp.n_emit, pp.n_work, pp.n_prefill_work, pp.n_deltas, pp.n_prompts) == (4, 4, 4, 4, 0, 4, 0)
    d = pp.data
    assert d[:20].tolist() == [2, 40, 1, 0, 0, 1, 31, 1, 1, 1, 50, 0, 1, 2, 2, 50, 0, 1, 3, 3]
    assert d[20:28].tolist() == [0, 0, 1, 0, 2, 0, 3, 0]
    assert d[28:40].tolist() == [1, 2, 33, 50, 0, 900, 50, 0, 900, 50, 0, 900]
    assert d.size == 40 and pp.emit_ids == [7, 4] and pp.seq == 8
