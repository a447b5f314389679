"""Every reference citation in the repo points at real lines of the reference.

A citation is ``<module>.py:N`` or ``<module>.py:N-M`` for a module of the
reference package (``/root/reference/pkg/src/wavesweep``).  Each one must lie
inside the file, and the cited lines must contain at least one identifier
that the citing line names (the symbol or expression being cited), so an
offset citation -- lines taken from the wrong file, or from concatenated
files -- fails.  Runs where the reference is present (the build container).
"""

import os
import re
import subprocess

import pytest

REF = "/root/reference/pkg/src/wavesweep"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODULES = ("grid", "kernels", "sweep", "driver", "parallel", "bench", "oracles", "cli")
CITE = re.compile(r"(?<![\w/])(" + "|".join(MODULES) + r")\.py:(\d+)(?:-(\d+))?")
# documents written by others (survey, judge, advisor) are not checked here
SKIP = {"VERDICT.md", "SURVEY.md", "ADVICE.md", "BASELINE.md", "PAPERS.md", "SNIPPETS.md",
        "tests/test_citations.py"}
STOP = {"the", "and", "for", "with", "from", "reference", "line", "lines", "same", "order",
        "here", "this", "that", "each", "every", "side", "then", "into", "when", "only", "also",
        "first", "kernels", "driver", "sweep", "grid", "bench", "parallel", "oracle",
        "oracles", "numpy", "python", "def", "class", "return", "self", "none", "true", "false"}

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


def _sources():
    out = subprocess.run(["git", "ls-files"], cwd=ROOT, capture_output=True, text=True).stdout
    for f in out.split():
        if f in SKIP or f.startswith(("profiles/", "gpurun_out/", "baseline/")):
            continue
        if re.search(r"\.(py|md|h|cu|cuh|sh)$", f):
            yield f


def _citations():
    for f in _sources():
        lines = open(os.path.join(ROOT, f), encoding="utf-8").read().split("\n")
        for n, ln in enumerate(lines):
            for m in CITE.finditer(ln):
                # the citing context: this line and its neighbours (wrapped prose)
                ctx = " ".join(lines[max(0, n - 1):n + 2])
                yield f, n + 1, m.group(1), int(m.group(2)), int(m.group(3) or m.group(2)), ctx


CITES = list(_citations()) if os.path.isdir(REF) else []


def _ref_lines(mod):
    with open(os.path.join(REF, mod + ".py"), encoding="utf-8") as fh:
        return fh.read().split("\n")


def test_there_are_citations():
    assert len(CITES) > 100


def test_every_citation_is_inside_its_file():
    bad = []
    for f, n, mod, a, b, _ in CITES:
        L = _ref_lines(mod)
        if not (1 <= a <= b <= len(L)):
            bad.append(f"{f}:{n} cites {mod}.py:{a}-{b} (file has {len(L)} lines)")
    assert not bad, "\n".join(bad)


def _idents(text):
    return {w.lower() for w in re.findall(r"[A-Za-z_][A-Za-z0-9_]{2,}", text)} - STOP


def test_every_citation_names_something_in_the_cited_lines():
    bad = []
    for f, n, mod, a, b, ctx in CITES:
        L = _ref_lines(mod)
        cited = " ".join(L[a - 1:b])
        ctx_ids = _idents(CITE.sub(" ", ctx))
        if not ctx_ids & _idents(cited):
            bad.append(f"{f}:{n} {mod}.py:{a}-{b}: {L[a - 1].strip()[:60]!r}")
    assert not bad, f"{len(bad)} citations share no identifier with the cited lines:\n" + \
        "\n".join(bad)


@pytest.mark.parametrize("cite,symbol", [
    ("kernels.py:44-55", "class KernelError"), ("kernels.py:89-96", "DESCRIPTORS"),
    ("kernels.py:163-178", "def rp_advection"), ("kernels.py:181-213", "def rp_acoustics_const"),
    ("kernels.py:216-261", "def rp_acoustics_var"), ("kernels.py:264-340", "def rp_euler"),
    ("kernels.py:343-371", "def euler_flux"), ("kernels.py:374-393", "class Kernel"),
    ("kernels.py:396-440", "def make_kernel"), ("driver.py:34-57", "def choose_dt"),
    ("driver.py:199-225", "def step"), ("driver.py:228-250", "def run"),
    ("grid.py:179-193", "def fill_ghost"), ("sweep.py:68-75", "class SweepError"),
    ("sweep.py:175-251", "def sweep"), ("sweep.py:254-280", "def apply_update"),
    ("bench.py:209-234", "def emit_csv"), ("bench.py:236-264", "def parse_csv"),
    ("parallel.py:267-293", "def for_each_unit"),
])
def test_boundary_anchor_lines(cite, symbol):
    # the anchors include/wavestep.h and INTEGRATION.md cite for each entry point
    mod, rng = cite.split(".py:")
    a, b = (int(x) for x in rng.split("-"))
    assert symbol in "\n".join(_ref_lines(mod)[a - 1:b])
