"""Native trace reader/writer (ks_trace_parse / ks_trace_write, host C++)
against the reference parser's golden vectors (tests/golden/
parse_golden.json.gz, made by tests/golden/make_parse_golden.py from
kernsim.trace.parse_trace) and against the golden corpus documents.

CPU tests: the reader is host code (trace.py:281-328 is host code in the
reference too); the library is loaded, no kernel is launched.
"""

from __future__ import annotations

import ast
import gzip
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2006_03318_b200 import errors
from paper_2006_03318_b200.columnar import ColumnarTrace, dump_trace_columns, load_trace_columns
from paper_2006_03318_b200.trace import document_to_object, parse_trace

GOLD = Path(__file__).resolve().parent / "golden"
CASES = json.load(gzip.open(GOLD / "parse_golden.json.gz"))
THREADS = [None, 1, 3, 64]


def _corpus():
    d = json.load(gzip.open(GOLD / "golden.json.gz"))
    return [(c["name"], json.dumps(ast.literal_eval(c["doc"]) if isinstance(c["doc"], str)
                                   else c["doc"])) for c in d["cases"]]


@pytest.mark.parametrize("threads", THREADS)
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_reader_matches_reference(case, threads):
    err = case.get("error")
    if err is None:
        ct = load_trace_columns(case["text"], threads=threads)
        doc = ct.to_document()
        assert document_to_object(doc) == case["doc"]
        assert doc.metadata == case["metadata"]
        assert [[e.id, e.start, e.duration] for e in doc.events] == case["events_ns"]
        return
    with pytest.raises(errors.KernsimError) as ei:
        load_trace_columns(case["text"], threads=threads)
    if err.startswith("<non-kernsim"):
        # the reference crashes with a non-KernsimError; we name it
        assert ei.value.name in ("Unsupported", "SchemaViolation")
        return
    assert ei.value.name == err, (ei.value, case.get("message"))
    if err == "OverlapViolation":
        assert sorted([ei.value.first_id, ei.value.second_id]) == case["ids"]
    if err == "SchemaViolation":
        assert ei.value.message == case["message"]


@pytest.mark.parametrize("threads", [None, 2, 16])
def test_corpus_documents_and_roundtrip(threads):
    for name, text in _corpus():
        ref = parse_trace(text)
        ct = load_trace_columns(text, threads=threads)
        assert ct.to_document() == ref, name
        text2 = dump_trace_columns(ct, threads=threads)
        assert load_trace_columns(text2, threads=threads).to_document() == ref, name
        assert parse_trace(text2.decode()) == ref, name


def test_columns_match_from_events():
    for name, text in _corpus():
        ref = parse_trace(text)
        ct = load_trace_columns(text, threads=4)
        want = ColumnarTrace.from_document(ref)
        for k in ("id", "kind", "lane", "start", "duration", "correlation", "sync_target",
                  "is_dtoh"):
            assert np.array_equal(getattr(ct.cols, k), getattr(want.cols, k)), (name, k)
        assert ct.cols.lanes == want.cols.lanes, name
        assert ct.names == want.names and np.array_equal(ct.name_id, want.name_id), name
        tag, tags = ct.marker_tags()
        wtag, wtags = want.marker_tags()
        assert tags == wtags and np.array_equal(tag, wtag), name


def test_writer_escapes_like_json_dumps():
    text = CASES[[c["name"] for c in CASES].index("name_2")]["text"]
    ct = load_trace_columns(text)
    out = dump_trace_columns(ct).decode()
    assert '"\\ud83d\\ude00"' in out
    assert json.loads(out)["events"][0]["name"] == "\U0001F600"


def test_large_synthetic_roundtrip_parallel():
    """~200k events through write -> parse with many threads: columns equal."""
    from paper_2006_03318_b200.workloads import ingest_document_columns

    ct = ingest_document_columns(200_000, seed=3)
    text = dump_trace_columns(ct, threads=8)
    for th in (1, 7, 32):
        back = load_trace_columns(text, threads=th)
        for k in ("id", "kind", "start", "duration", "correlation", "is_dtoh"):
            assert np.array_equal(getattr(back.cols, k), getattr(ct.cols, k)), (th, k)
        # lane indices are first-appearance order in the document: compare by text
        for k in ("lane", "sync_target"):
            a = np.array([str(x) for x in back.cols.lanes] + ["-"])[getattr(back.cols, k)]
            b = np.array([str(x) for x in ct.cols.lanes] + ["-"])[getattr(ct.cols, k)]
            assert np.array_equal(a, b), (th, k)
        assert [back.names[i] for i in back.name_id[:1000]] == [ct.names[i] for i in ct.name_id[:1000]]
        assert np.array_equal(back.m_start, ct.m_start) and np.array_equal(back.m_end, ct.m_end)
        assert [str(back.cols.lanes[i]) for i in back.m_lane] == [str(ct.cols.lanes[i]) for i in ct.m_lane]
        assert [back.layers[i] for i in back.m_layer] == [ct.layers[i] for i in ct.m_layer]


def _random_doc(rng, n_events, n_markers):
    """A random trace document dict with reference-legal events/markers and a
    mix of number spellings (ints, decimals, exponents, long floats, strings)."""
    import math

    def t_us(ns):
        style = rng.integers(0, 6)
        if style == 0 and ns % 1000 == 0:
            return ns // 1000
        if style == 1:
            return ns / 1000
        if style == 2:
            return f"{ns / 1000:.6f}"            # Decimal string
        if style == 3:
            return float(f"{ns / 1000:.17g}")    # long float repr
        if style == 4:
            return float(f"{ns:.6e}") / 1000
        return ns / 1000
    lanes = ["cpu:0", "cpu:1", "gpu:0:7", "gpu:0:8", "comm:ring0"]
    names = ["cudaLaunchKernel", "sgemm_x", "memcpy_dtoh_async", "q\"uote", "unié", "tab\tx"]
    t = {ln: 0 for ln in lanes}
    ev = []
    corr = 1
    for i in range(n_events):
        ln = lanes[int(rng.integers(0, len(lanes)))]
        if ln.startswith("cpu"):
            kind = ["CpuApi", "CpuOther", "DataLoad", "Sync"][int(rng.integers(0, 4))]
        elif ln.startswith("gpu"):
            kind = ["GpuKernel", "GpuMemcpy"][int(rng.integers(0, 2))]
        else:
            kind = "Comm"
        start = t[ln] + int(rng.integers(0, 5000))
        dur = int(rng.integers(0, 9000))
        t[ln] = start + dur
        e = {"id": i * 3 + 1, "kind": kind, "name": names[int(rng.integers(0, len(names)))],
             "lane": ln, "start": t_us(start), "duration": t_us(dur)}
        if kind.startswith("Gpu") or rng.random() < 0.3:
            e["correlation"] = corr
            corr += 1
        if kind == "Sync" and rng.random() < 0.5:
            e["sync_target"] = "gpu:0:7"
        if rng.random() < 0.1:
            e["size_bytes"] = int(rng.integers(0, 1 << 40))
        if rng.random() < 0.1:
            e["extra"] = {"nested": [1, {"x": "}]"}]}
        ev.append(e)
    mk = []
    for j in range(n_markers):
        a = int(rng.integers(0, 10 ** 7))
        mk.append({"layer": f"l{j}", "phase": ["Forward", "Backward", "WeightUpdate"][j % 3],
                   "cpu_lane": "cpu:0", "start": t_us(a), "end": t_us(a + 1 + int(rng.integers(0, 10 ** 5)))})
    return {"schema_version": 1, "time_unit": "microseconds", "events": ev, "layer_markers": mk,
            "metadata": {"k": "v"}}


@pytest.mark.parametrize("seed", range(12))
def test_random_documents_match_python_parser(seed):
    """Native reader == the Python parse_trace mirror (pinned on the reference's
    vectors) on random documents, compact and indented, 1 and 13 threads."""
    rng = np.random.default_rng(seed)
    doc = _random_doc(rng, int(rng.integers(0, 3000)), int(rng.integers(0, 40)))
    for text in (json.dumps(doc), json.dumps(doc, indent=int(rng.integers(0, 4)))):
        try:
            want = parse_trace(text)
        except errors.KernsimError as e:
            with pytest.raises(errors.KernsimError) as ei:
                load_trace_columns(text, threads=13)
            assert ei.value.name == e.name
            continue
        for th in (1, 13):
            assert load_trace_columns(text, threads=th).to_document() == want
        back = load_trace_columns(dump_trace_columns(load_trace_columns(text)), threads=5)
        assert back.to_document() == want
