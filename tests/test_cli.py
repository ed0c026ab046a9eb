"""The `turnip` CLI is flag- and exit-code-compatible with the reference
`memplan` CLI (proj/tools/memplan_main.cpp): the reference's own CLI test
script (proj/tests/cli_test.sh) is run against it when the reference is
present; a self-contained subset always runs."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2405_16283_b200", "lib", "turnip")
REF_CLI_TEST = "/root/reference/proj/tests/cli_test.sh"


def run(*args, **kw):
    return subprocess.run([BIN, *args], capture_output=True, text=True, **kw)


def test_reference_cli_script(tmp_path):
    if not os.path.exists(REF_CLI_TEST):
        pytest.skip("reference sources not present (GPU box)")
    r = subprocess.run(["bash", REF_CLI_TEST, BIN, str(tmp_path / "work")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all CLI checks passed" in r.stdout


def test_cli_exit_codes_and_compile(tmp_path):
    g = tmp_path / "mm3.json"
    assert run("gen", "--kind", "matmul", "--parts", "3", "--out", str(g)).returncode == 0
    r = run("validate", "--graph", str(g))
    assert r.returncode == 0 and r.stdout.strip() == "ok"
    assert run("validate").returncode == 2
    assert run("validate", "--graph", str(tmp_path / "missing.json")).returncode == 2
    r = run("compile", "--graph", str(g), "--capacities", "slots:5", "--out", str(tmp_path / "m.json"))
    st = json.loads(r.stdout)
    assert r.returncode == 0 and st["memory_edges"] == 2 and st["required_memory_edges"] == 1
    r = run("verify", "--graph", str(g), "--memgraph", str(tmp_path / "m.json"), "--schedules", "100")
    assert r.returncode == 0 and json.loads(r.stdout)["all_passed"]
    bad = json.loads(open(tmp_path / "m.json").read())
    bad["edges"] = [e for e in bad["edges"] if not (e["kind"] == "memory" and not e["superfluous"])]
    (tmp_path / "bad.json").write_text(json.dumps(bad))
    assert run("verify", "--graph", str(g), "--memgraph", str(tmp_path / "bad.json")).returncode == 1
    assert run("bogus").returncode == 2
