"""The compact marching-cubes table (include/wfk_mc_cases.h) equals the
reference's kMcTriTable (proj/src/mc_tables.cpp) entry for entry.  Runs where
/root/reference is mounted (the build container); skipped elsewhere."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj/src/mc_tables.cpp"


def ours():
    txt = open(os.path.join(ROOT, "include", "wfk_mc_cases.h")).read()
    body = txt[txt.index("kWfMcCases[256]"):txt.index("kWfMcEdgeCorners")]
    cases = re.findall(r'"([0-9a-b]*)"', body)
    assert len(cases) == 256
    return [[int(c, 16) for c in s] for s in cases]


def test_case_table_shape():
    t = ours()
    assert t[0] == [] and t[255] == []
    assert all(len(c) % 3 == 0 and len(c) <= 15 for c in t)
    assert all(0 <= e < 12 for c in t for e in c)


@pytest.mark.skipif(not os.path.exists(REF), reason="reference not mounted")
def test_matches_reference_table():
    src = open(REF).read()
    body = src[src.index("kMcTriTable"):src.index("kMcEdgeCorners")]
    rows = re.findall(r"\{([-0-9, ]+)\}", body)
    ref = []
    for r in rows:
        v = [int(x) for x in r.split(",")]
        ref.append(v[: v.index(-1)] if -1 in v else v)
    assert ref == ours()
