"""Router-dump format: writer/reader round trips and validation on
the CPU; streamed ingestion vs in-memory ingestion on the GPU."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2605_19945_b200 import routerdump as rd
from paper_2605_19945_b200.errors import ValidationError


def _ids(rng, L, N, k, E, dtype=np.int16):
    return rng.integers(0, E, (L, N, k)).astype(dtype)


@pytest.mark.parametrize("id_bytes", [2, 4])
def test_roundtrip_uneven_appends(tmp_path, id_bytes):
    rng = np.random.default_rng(1)
    L, k, E, B, S = 3, 4, 40, 16, 5  # 80 tokens per chunk
    dt = np.int16 if id_bytes == 2 else np.int32
    parts = [_ids(rng, L, n, k, E, dt) for n in (7, 100, 1, 33, 59)]  # 200 tokens: 2 full chunks + 40
    path = tmp_path / "r.gemr"
    with rd.RouterDumpWriter(path, L, k, E, tokens_per_step=B, chunk_steps=S, id_bytes=id_bytes) as w:
        for p in parts:
            w.append(p)
    d = rd.RouterDump(path)
    h = d.header
    assert (h.num_layers, h.top_k, h.num_experts, h.tokens_per_step, h.chunk_steps, h.num_tokens, h.id_bytes) == \
        (L, k, E, B, S, 200, id_bytes)
    assert h.num_chunks == 3 and h.num_steps == 13
    want = np.concatenate(parts, axis=1)
    assert np.array_equal(d.all_ids(), want)
    assert [d.chunk(c).shape[1] for c in range(3)] == [80, 80, 40]
    buf = np.zeros(L * 80 * k, dtype=dt)
    n = d.read_chunk_into(2, buf)
    assert n == L * 40 * k and np.array_equal(buf[:n].reshape(L, 40, k), want[:, 160:])


def test_rejects_bad_files(tmp_path):
    p = tmp_path / "x.gemr"
    p.write_bytes(b"NOTADUMP" + bytes(56))
    with pytest.raises(ValidationError, match="magic"):
        rd.RouterDump(p)
    p.write_bytes(b"GEMR")
    with pytest.raises(ValidationError, match="truncated"):
        rd.RouterDump(p)
    w = rd.RouterDumpWriter(p, 2, 2, 8, tokens_per_step=4, chunk_steps=2)
    w.append(np.zeros((2, 20, 2), dtype=np.int16))
    w.close()
    raw = p.read_bytes()
    p.write_bytes(raw[:-6])  # cut the last ids
    with pytest.raises(ValidationError, match="holds"):
        rd.RouterDump(p)
    with pytest.raises(ValidationError, match="shape"):
        rd.RouterDumpWriter(tmp_path / "y.gemr", 2, 2, 8).append(np.zeros((3, 4, 2), dtype=np.int16))
    with pytest.raises(ValidationError, match="id_bytes"):
        rd.RouterDumpWriter(tmp_path / "z.gemr", 2, 2, 8, id_bytes=1)


def test_header_layout_is_fixed():
    h = rd.DumpHeader(2, 94, 8, 128, 1024, 64, 1 << 24)
    raw = h.pack()
    assert len(raw) == 64 and raw[:8] == b"GEMRDMP1"
    assert rd.DumpHeader.unpack(raw) == h
    assert h.chunk_offset(3) == 64 + 3 * 94 * 64 * 1024 * 8 * 2


@pytest.mark.gpu
@pytest.mark.parametrize("id_bytes,N,S", [(2, 37 * 64 + 17, 7), (4, 20 * 64, 4), (2, 64 * 64, 64)])
def test_stream_statistics_equals_in_memory(tmp_path, id_bytes, N, S):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2605_19945_b200 import ingest

    rng = np.random.default_rng(N)
    L, k, E, B = 3, 8, 64, 64
    dt = np.int16 if id_bytes == 2 else np.int32
    ids = np.stack([np.stack([rng.choice(E, k, replace=False) for _ in range(N)]) for _ in range(L)]).astype(dt)
    path = tmp_path / "s.gemr"
    with rd.RouterDumpWriter(path, L, k, E, tokens_per_step=B, chunk_steps=S, id_bytes=id_bytes) as w:
        for a in range(0, N, 500):
            w.append(ids[:, a:a + 500])
    got = rd.stream_statistics(path)
    want = ingest.trace_statistics(torch.from_numpy(ids).cuda(), B, E)
    torch.cuda.synchronize()
    for name in ("hist", "colsum", "active", "heavy", "dropped"):
        assert torch.equal(getattr(got.hist, name), getattr(want.hist, name)), name
    assert torch.equal(got.gram, want.gram)
    assert torch.equal(got.mean_utilization, want.mean_utilization)
    assert torch.equal(got.classes.cls, want.classes.cls) and torch.equal(got.classes.group, want.classes.group)


@pytest.mark.gpu
def test_cli_ingest_then_multi_layer(tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import json

    import paper_2605_19945_b200 as gem
    from oracle import oracle as orc
    from paper_2605_19945_b200 import cli, ingest

    L, N, k, E, B = 2, 64 * 40, 8, 32, 64
    spec = ingest.TopkTraceSpec(num_layers=L, num_tokens=N, top_k=k, num_experts=E, tokens_per_step=B, seed=4)
    w, role = ingest.planted_layout(spec)
    ids = orc.gen_topk(L, N, k, B, E, w, role, ingest._prob_u32(spec.consistent_probability),
                       ingest._prob_u32(spec.burst_probability), spec.burst_multiplier, spec.seed)
    dump = tmp_path / "router.gemr"
    with rd.RouterDumpWriter(dump, L, k, E, tokens_per_step=B, chunk_steps=16) as wr:
        wr.append(ids)
    out = tmp_path / "traces"
    assert cli.main(["ingest", "--dump", str(dump), "--output-dir", str(out), "--quiet"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["result"]["num_tokens"] == N and len(rep["result"]["layers"]) == L
    hist, _ = orc.topk_hist(ids, B, E)
    for l in range(L):
        tr = gem.load_trace(out / f"layer{l:02d}.json")
        assert np.array_equal(tr.tokens, hist[l])
        cls, grp = orc.classify(hist[l])
        got = rep["result"]["layers"][l]
        assert got["consistent"] == [e for e in range(E) if cls[e] == 1]
    prof = tmp_path / "p.json"
    assert cli.main(["gen-profile", "--gpus", "4", "--setup", "moderate", "--seed", "1", "--output", str(prof),
                     "--quiet"]) == 0
    assert cli.main(["multi-layer", "--trace-dir", str(out), "--profile", str(prof), "--output-dir",
                     str(tmp_path / "maps"), "--seed", "0", "--restarts", "3", "--quiet"]) == 0
    assert len(list((tmp_path / "maps").glob("*.mapping.json"))) == L
