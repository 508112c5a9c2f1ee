"""migrate-plan: same JSON as the reference CLI (golden stdout from
`tpsim migrate-plan`, tests/golden) and the reference test_cli.py checks."""

import json

import pytest

from paper_2605_05467_b200.cli import main


def _write(tmp_path, doc):
    p = tmp_path / "layout.json"
    p.write_text(json.dumps(doc))
    return p


def test_migrate_plan_matches_reference_output(tmp_path, capsys, ref_golden):
    g = ref_golden["cli"]
    out = tmp_path / "plan.json"
    rc = main(["migrate-plan", "--layout", str(_write(tmp_path, g["layout"])), "--new-tp", "2",
               "--out", str(out)])
    assert rc == g["rc"] == 0
    assert json.loads(out.read_text()) == g["stdout"]
    assert json.loads(capsys.readouterr().out) == g["stdout"]


def test_migrate_plan_tp_mismatch_exits_2(tmp_path, capsys, ref_golden):
    rc = main(["migrate-plan", "--layout", str(_write(tmp_path, ref_golden["cli"]["layout"])),
               "--new-tp", "4"])
    assert rc == 2
    assert "new_tp" in capsys.readouterr().err


def test_migrate_plan_bad_layout_exits_2(tmp_path, capsys):
    doc = {"total_heads": 8, "groups": [{"gpus": [1, 2, 3], "requests": []}]}
    rc = main(["migrate-plan", "--layout", str(_write(tmp_path, doc)), "--new-tp", "3"])
    assert rc == 2
    assert "divisible" in capsys.readouterr().err


def test_missing_file_exits_2(tmp_path, capsys):
    assert main(["migrate-plan", "--layout", str(tmp_path / "nope.json"), "--new-tp", "2"]) == 2


@pytest.mark.gpu
def test_migrate_plan_execute(tmp_path, capsys):
    doc = {"total_heads": 8, "kv_bytes_per_token_per_head": 16384,
           "groups": [{"gpus": [0], "requests": [{"id": 0, "context_len": 512}, {"id": 2, "context_len": 77}]},
                      {"gpus": [1], "requests": [{"id": 1, "context_len": 300}]}]}
    rc = main(["migrate-plan", "--layout", str(_write(tmp_path, doc)), "--new-tp", "2", "--execute",
               "--fragmented"])
    assert rc == 0
    res = json.loads(capsys.readouterr().out)
    m = res["measured"]
    assert m["bit_exact_property"] and m["placement_matches_reference"]
    assert m["bytes"] == res["total_bytes"]
