"""K2b token-level co-selection counts against the oracle.

The reference has no co-selection statistic (its only co-activation measure is
the step-level Pearson, /root/reference/pkg/src/gemap/trace.py:100-113), so the
oracle is the definition restated (oracle.coselect: OᵀO of the 0/1 selection
indicator, and oracle.coselect_loops: explicit per-token pair loops), tied to
the pinned ingestion path by diag(C) == K1's colsum for distinct router ids.
Integer counts: bit-exact everywhere.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")


# ------------------------------------------------------------------ CPU: oracle

def test_oracle_definitions_agree(oracle):
    rng = np.random.default_rng(5)
    ids = rng.integers(-2, 19, (2, 300, 6)).astype(np.int16)  # dropped ids and in-token repeats
    a, b = oracle.coselect(ids, 17), oracle.coselect_loops(ids, 17)
    assert np.array_equal(a, b)
    assert np.array_equal(a, a.transpose(0, 2, 1))


def test_oracle_diag_is_colsum_for_distinct_ids(oracle):
    rng = np.random.default_rng(6)
    E, k = 40, 8
    ids = np.stack([np.stack([rng.permutation(E)[:k] for _ in range(500)]) for _ in range(2)]).astype(np.int32)
    c = oracle.coselect(ids, E)
    hist, _ = oracle.topk_hist(ids, 50, E)
    assert np.array_equal(np.diagonal(c, axis1=1, axis2=2), hist.sum(axis=1))
    # every token contributes k*k ordered pairs
    assert np.array_equal(c.sum(axis=(1, 2)), np.full(2, 500 * k * k))


# ------------------------------------------------------------------ GPU: parity

gpu = pytest.mark.gpu


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2605_19945_b200 import ingest

    return ingest


def _distinct_ids(rng, L, N, k, E, dtype):
    keys = rng.random((L, N, E))
    return np.argsort(keys, axis=2)[:, :, :k].astype(dtype)


SHAPES = [  # L, N, k, E, dtype, distinct
    (2, 1000, 8, 128, np.int16, True),      # tensor cores, E = 128, 16-byte tokens
    (3, 777, 8, 128, np.int32, True),       # 32-byte tokens, ragged N
    (1, 4096, 8, 256, np.int16, True),      # two expert blocks (128x256 + 128x128 MMAs)
    (2, 2048, 8, 200, np.int16, False),     # padded second block, repeats and dropped ids
    (3, 2048, 2, 8, np.int16, True),        # Mixtral k=2: scalar token path
    (2, 1024, 8, 64, np.int32, False),      # OLMoE-like E, padded rows
    (5, 300, 8, 128, np.int16, True),       # many layer segments per CTA
    (1, 1000, 8, 300, np.int16, True),      # E > 256: scatter kernel
    (2, 999, 3, 50, np.int16, False),       # N*k*2 % 16 != 0: scatter kernel
]


@gpu
@pytest.mark.parametrize("L,N,k,E,dtype,distinct", SHAPES)
def test_coselect_matches_oracle(oracle, L, N, k, E, dtype, distinct):
    ingest = _cuda()
    rng = np.random.default_rng(L * 1000 + N + E)
    ids = _distinct_ids(rng, L, N, k, E, dtype) if distinct else rng.integers(-3, E + 3, (L, N, k)).astype(dtype)
    want = oracle.coselect(ids, E)
    dev = torch.from_numpy(ids).cuda()
    got = ingest.token_coselection(dev, E)
    assert np.array_equal(got.cpu().numpy(), want)
    sc = ingest.token_coselection(dev, E, path="scatter")
    assert np.array_equal(sc.cpu().numpy(), want)
    if distinct:
        hist, _ = oracle.topk_hist(ids, 64, E)
        assert np.array_equal(np.diagonal(got.cpu().numpy(), axis1=1, axis2=2), hist.sum(axis=1))


@gpu
def test_coselect_paths_and_accumulation(oracle):
    ingest = _cuda()
    rng = np.random.default_rng(11)
    ids = torch.from_numpy(_distinct_ids(rng, 2, 4096, 8, 128, np.int16)).cuda()
    assert ingest.coselection_path(ids, 128) == "tc"
    assert ingest.coselection_path(ids, 300) == "scatter"
    odd = ids.reshape(-1)[1:1 + 2 * 4095 * 8].view(2, 4095, 8)  # 2-byte offset: not 16-byte aligned
    assert ingest.coselection_path(odd, 128) == "scatter"
    assert np.array_equal(ingest.token_coselection(odd, 128).cpu().numpy(), oracle.coselect(odd.cpu().numpy(), 128))
    out = ingest.token_coselection(ids, 128)
    ingest.token_coselection(ids, 128, out=out)  # accumulates
    assert np.array_equal(out.cpu().numpy(), 2 * oracle.coselect(ids.cpu().numpy(), 128))


@gpu
def test_coselect_in_statistics_phase_on_benchmark_trace(oracle):
    """The statistics phase with coselect=True on the benchmark's own generator
    (Qwen3-235B shape, a few hundred steps): OᵀO == oracle, diag == colsum."""
    ingest = _cuda()
    spec = ingest.TopkTraceSpec(num_layers=3, num_tokens=300 * 1024, top_k=8, num_experts=128, seed=0)
    ids = ingest.generate_topk_ids(spec)
    st = ingest.trace_statistics(ids, 1024, 128, coselect=True).check()
    cs = st.hist.stats.coselect.cpu().numpy()
    assert np.array_equal(cs, oracle.coselect(ids.cpu().numpy(), 128))
    assert np.array_equal(np.diagonal(cs, axis1=1, axis2=2), st.hist.colsum.cpu().numpy())
