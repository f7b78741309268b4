"""Generated / duplicated tables stay in sync (CPU only)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_log_table_is_what_the_generator_writes(tmp_path):
    """csrc/esdg_log_table.inc is committed; tools/gen_log_table.py must
    reproduce it bit for bit (hex float literals)."""
    pytest.importorskip("mpmath")
    out = tmp_path / "table.inc"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_log_table.py"), str(out)],
                   check=True, capture_output=True)
    committed = open(os.path.join(ROOT, "paper_2605_16684_b200", "csrc", "esdg_log_table.inc")).read()
    assert out.read_text() == committed


def test_log_table_properties():
    """The properties log_pos relies on (esdg_log.cuh): 128 rows, log c hi a
    multiple of 2^-43, interval 80 is c = 1 exactly, its neighbours carry a
    1/c with at most 9 significant bits."""
    rows, ln2 = [], None
    for line in open(os.path.join(ROOT, "paper_2605_16684_b200", "csrc", "esdg_log_table.inc")):
        if line.startswith("ESDG_LOG_ROW("):
            rows.append([float.fromhex(x.strip()) for x in line[len("ESDG_LOG_ROW("):-2].split(",")])
        elif line.startswith("ESDG_LOG_LN2("):
            ln2 = [float.fromhex(x.strip()) for x in line[len("ESDG_LOG_LN2("):-2].split(",")]
    assert len(rows) == 128 and ln2 is not None
    assert (ln2[0] * 2.0 ** 43).is_integer() and abs(ln2[0] + ln2[1] - 0.6931471805599453) < 1e-16
    for invc, hi, lo in rows:
        assert (hi * 2.0 ** 43).is_integer()
        assert abs(lo) <= 2.0 ** -44
    assert rows[80] == [1.0, 0.0, 0.0]
    for i in list(range(72, 80)) + list(range(81, 85)):
        assert (rows[i][0] * 256).is_integer(), i


def test_work_models_agree():
    """bench.py and the runner quote the same PerfRecord model
    (diagnostics.cpp:33-81)."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2605_16684_b200 import runner
    for nq in range(2, 9):
        for rb in (4, 8):
            b, r = bench.work_model(nq, rb), runner.work_model(nq, rb)
            assert (b["volume_flops"], b["volume_bytes"]) == r["volume"]
            assert (b["surface_flops"], b["surface_bytes"]) == r["surface"]
            assert b["update_bytes"] == r["update"][1]


def test_yperm_tables_are_permutations():
    """csrc/esdg_yperm_tables.inc (tools/yperm_search.py): every table assigns each y
    line of its tile to exactly one thread."""
    import re
    path = os.path.join(ROOT, "paper_2605_16684_b200", "csrc", "esdg_yperm_tables.inc")
    text = open(path).read()
    tables = re.findall(r"c_yperm_(\d+)_(\d+)_(\d+)\[(\d+)\] = \{([^}]*)\}", text)
    assert len(tables) >= 4
    for nq, nbytes, epb, n, body in tables:
        vals = [int(v) for v in body.replace("\n", " ").split(",") if v.strip()]
        assert len(vals) == int(n) == int(epb) * int(nq) ** 2
        assert sorted(vals) == list(range(int(n)))
