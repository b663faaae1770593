"""GPU: the §8(f) rows beside the path — batch driver (cli.cpp:164-210,
RunReport JSON cli.cpp:93-107, criterion 11 determinism) and the LEQT
equality-table container with real ciphertexts (preprocess.cpp:80-194)."""
import io
import json

import pytest

import paper_2508_14568_b200 as L

pytestmark = pytest.mark.gpu


def test_batch_lines_match_reference_reports(golden):
    cases = [c for c in golden["cases"]
             if "report" in c and c["mode"] == "exact" and c["encoding"] == "ascii7"
             and c["budget"] == 4000.0 and c["key_encoding"] == "negated" and not c["preprocess"]]
    assert len(cases) >= 10
    lines = [json.dumps({"a": c["a"], "b": c["b"]}) for c in cases]
    lines.insert(1, "{not json")
    lines.insert(3, json.dumps({"a": "x"}))
    lines.insert(5, json.dumps({"a": "abc", "b": "abé"}))  # outside ascii7
    out = L.run_batch(lines)
    assert len(out) == len(lines)
    assert "bad JSON" in json.loads(out[1])["error"]
    assert "needs string fields" in json.loads(out[3])["error"]
    assert "alphabet" in json.loads(out[5])["error"]
    got = [json.loads(o) for i, o in enumerate(out) if i not in (1, 3, 5)]
    for rep, case in zip(got, cases):
        assert list(rep.keys()) == L.leuven.REPORT_FIELDS
        for k in L.leuven.REPORT_FIELDS:
            assert rep[k] == (case["report"][k] if k != "mode" else "exact"), (case["a"], k)
    assert L.run_batch(lines) == out  # byte-identical on rerun (criterion 11)


def test_eq_table_container_roundtrip():
    ctx = L.Context(seed=0)
    spec = L.AlphabetSpec.lower26()
    xs = L.encrypt_string("abbey", spec, ctx)
    table, pbs = L.build_eq_table(ctx, xs, spec)
    assert pbs == 2 * 26 * 5
    buf = io.BytesIO()
    n = L.save_eq_table(table, buf)
    assert n > 26 * 5 * 2049 * 8
    loaded = L.load_eq_table(ctx, io.BytesIO(buf.getvalue()))
    assert loaded.string_length() == 5 and loaded.subset() == spec.charset()
    for ch in "abcey":
        for i in range(1, 6):
            assert ctx.decrypt([loaded.lookup(ch, i)])[0] == ctx.decrypt([table.lookup(ch, i)])[0]
    assert ctx.export([loaded.lookup("b", 2)]).tobytes() == ctx.export([table.lookup("b", 2)]).tobytes()
    r1 = L.distance_preprocessed(ctx, table, "abbes", L.BandSpec.exact(5, 5))
    r2 = L.distance_preprocessed(ctx, loaded, "abbes", L.BandSpec.exact(5, 5))
    assert ctx.decrypt([r1.score])[0] == ctx.decrypt([r2.score])[0] == 1
    data = buf.getvalue()
    with pytest.raises(L.FormatError):
        L.load_eq_table(ctx, io.BytesIO(b"XXXX" + data[4:]))
    with pytest.raises(L.FormatError):
        L.load_eq_table(ctx, io.BytesIO(data[: len(data) // 2]))
    other = L.Context(seed=99)
    with pytest.raises(L.InvalidParams):
        L.load_eq_table(other, io.BytesIO(data))
    other.close()


def test_cli_compute_and_batch(tmp_path, golden):
    import io as _io
    from paper_2508_14568_b200.__main__ import main
    case = next(c for c in golden["cases"] if c["a"] and c["b"] and "report" in c
                and c["mode"] == "exact" and c["encoding"] == "ascii7"
                and c["budget"] == 4000.0 and c["key_encoding"] == "negated" and not c["preprocess"])
    out = _io.StringIO()
    assert main(["compute", "--a", case["a"], "--b", case["b"], "--json"], out=out) == 0
    rep = json.loads(out.getvalue())
    assert rep["distance"] == case["report"]["distance"] and "wall_time_ms" in rep
    p = tmp_path / "in.jsonl"
    p.write_text(json.dumps({"a": case["a"], "b": case["b"]}) + "\n")
    out = _io.StringIO()
    assert main(["batch", "--input", str(p), "--threads", "4"], out=out) == 0
    assert json.loads(out.getvalue())["pbs_total"] == case["report"]["pbs_total"]
    err = _io.StringIO()
    assert main(["compute", "--a", "abcdef", "--b", "a", "--mode", "approx", "--ell", "1"],
                out=_io.StringIO(), err=err) == 3


def test_preprocessed_batch_database_scan(ctx):
    """One preprocessed encrypted query against many plaintext strings in one
    wavefront equals the per-string distance_preprocessed (distance and every
    counter) and Wagner-Fischer."""
    from paper_2508_14568_b200 import workloads as W
    a, b = W.cfg4()
    a = a[:24]
    spec = L.AlphabetSpec.dna4()
    xs = L.encrypt_string(a, spec, ctx)
    table, _ = L.build_eq_table(ctx, xs, spec)
    plains = [b[:20], a, W.mutate(a, 3, W.MT19937(77), draw=W.dna), "ACGT", "", "T" * 30]
    bands = [L.BandSpec.exact(len(a), len(p)) for p in plains]
    runs = L.distance_preprocessed_batch(ctx, table, plains, bands)
    got = ctx.decrypt([r.score for r in runs])
    for p, band, r, d in zip(plains, bands, runs, got):
        one = L.distance_preprocessed(ctx, table, p, band)
        assert d == ctx.decrypt([one.score])[0] == L.wf_distance(a, p) % 32, p
        assert (r.visited_cells, r.equality_pbs, r.kernel_pbs, r.refreshes, r.max_key_variance) == (
            one.visited_cells, one.equality_pbs, one.kernel_pbs, one.refreshes, one.max_key_variance)
    with pytest.raises(L.CharNotInSubset):
        L.distance_preprocessed_batch(ctx, table, ["ACGX"], [L.BandSpec.exact(len(a), 4)])
