"""The slab planner's host layout (paper_2311_07710_b200/csrc/slab_layout.cpp)
on the CPU: tests/slab_layout_check.cpp is compiled together with the
planner's source and checks, over synthetic run lengths of several shapes and
every row order, that the tiles, offsets and metadata place each (window,
W row) run exactly once in the form slab.cuh reads them (rows sorted by run
inside a tile, slice offsets, 8-aligned metadata with zeroed padding, the
metadata written completely into a caller-provided buffer). The layout must
not depend on the number of planner threads: the runs with 1 and 4 threads
print the same hashes."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "..", "paper_2311_07710_b200", "csrc")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    exe = str(tmp_path_factory.mktemp("slab_layout") / "slab_layout_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, os.path.join(HERE, "slab_layout_check.cpp"),
                    os.path.join(CSRC, "slab_layout.cpp"), "-lpthread", "-o", exe], check=True)
    return exe


def run(exe, threads):
    env = dict(os.environ, RAPDHG_PLAN_THREADS=str(threads))
    env.pop("RAPDHG_TRACE", None)
    p = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    lines = p.stdout.split("\n")
    lines = [ln for ln in lines if ln]
    assert lines and all(ln.startswith("OK ") for ln in lines), p.stdout
    return lines


def test_layout_invariants_and_thread_independence(checker):
    one = run(checker, 1)
    four = run(checker, 4)
    assert one == four
    # the caller's buffer (pinned staging in slab.cu) gets the same metadata
    # as the planner's own vector
    by_case = {}
    for ln in one:
        _, *name, _, order, _, sink, h = ln.split()
        by_case.setdefault((" ".join(name), order), set()).add(h)
    assert all(len(hs) == 1 for hs in by_case.values())
    assert len(by_case) == 7 * 3
