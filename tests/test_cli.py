"""The `turnip` CLI keeps the reference `memplan` CLI's flags and exit codes
(proj/tools/memplan_main.cpp) for the subcommands around the execute path;
the toy `gen` subcommand is out of scope, so the reference's
cli_test.sh (which starts with `gen`) is not run against it."""
import json
import os
import subprocess

import pytest

from corpus import taskgraph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2405_16283_b200", "lib", "turnip")


def run(*args, **kw):
    return subprocess.run([BIN, *args], capture_output=True, text=True, **kw)


def test_cli_exit_codes_and_compile(tmp_path):
    g = tmp_path / "mm3.json"
    g.write_text(taskgraph("gen_matmul", [3]))
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
