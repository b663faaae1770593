"""CPU: the plaintext side of the reference's Python/CLI surface
(bindings/module.cpp:47-108, cli.cpp:212-238) against the compiled
reference's golden outputs: the product's own lookup tables (lut_dump /
`table`), eq_cost / `eqcost`, banded_distance."""
import io

import pytest

import paper_2508_14568_b200 as L
from paper_2508_14568_b200.__main__ import main


def test_product_tables_equal_reference(golden):
    luts = golden["luts"]
    assert L.lut_table("minlut-original") == luts["minlut-original"]
    assert L.lut_table("minlut-negated") == luts["minlut-negated"]
    assert L.lut_table("eqlut") == luts["eqlut1"]
    assert L.lut_table("eqlut9") == luts["eqlut9"]
    dump = L.lut_dump("minlut-negated").splitlines()
    assert len(dump) == 16 and dump[3] == "3\t1"
    with pytest.raises(L.InvalidParams):
        L.lut_table("nosuch")


def test_eq_cost_equals_reference(golden):
    for tech, want in golden["eq_cost"].items():
        assert [L.eq_cost(tech, b) for b in range(1, 65)] == want, tech
    with pytest.raises(L.OutOfRangeValue):
        L.eq_cost("combined", 0)
    with pytest.raises(L.InvalidParams):
        L.eq_cost("nosuch", 4)


def test_banded_distance_equals_reference(golden):
    for case in golden["banded"]:
        if case["error"] is None:
            assert L.banded_distance(case["a"], case["b"], case["half_width"]) == case["distance"]
        else:
            with pytest.raises(L.BandTooNarrow):
                L.banded_distance(case["a"], case["b"], case["half_width"])


def test_cli_table_and_eqcost(golden):
    out = io.StringIO()
    assert main(["table", "eqlut9"], out=out) == 0
    assert out.getvalue().splitlines()[0] == "0\t9"
    assert main(["table", "nosuch"], out=io.StringIO(), err=io.StringIO()) == 2
    out = io.StringIO()
    assert main(["eqcost", "--max-bits", "8"], out=out) == 0
    rows = out.getvalue().splitlines()
    assert rows[0] == "bits,standard,ours,combined" and len(rows) == 9
    b, std, ours, comb = (int(x) for x in rows[7].split(","))
    assert (std, ours, comb) == tuple(golden["eq_cost"][t][b - 1]
                                      for t in ("standard_2bit", "ours_4bit", "combined"))
