"""INTEGRATION.md's reference-side binding, executed verbatim: its python
block becomes hrgen/_b200.py of a scratch package (whose graph.Graph is the
CSR Graph of hrgen graph.py:15-81, here the package's mirror), bound to the
built libhrgen_b200.so, and its graph must equal the package's generate()."""

import os
import re
import sys
import textwrap

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def stub_source():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    stub = [b for b in blocks if b.startswith("# hrgen/_b200.py")]
    assert len(stub) == 1
    return stub[0]


def test_stub_parses_and_declares_every_call():
    src = stub_source()
    compile(src, "hrgen/_b200.py", "exec")
    called = set(re.findall(r"_L\.(hrg_[a-z_]+)\(", src))
    declared = set(re.findall(r'\("(hrg_[a-z_]+)", ', src))
    assert called <= declared, called - declared


@pytest.mark.gpu
def test_stub_generates_the_graph(tmp_path, monkeypatch):
    import paper_1501_03545_b200 as P
    pkg = tmp_path / "hrgen_scratch"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "graph.py").write_text(textwrap.dedent("""
        from paper_1501_03545_b200.graph import Graph  # hrgen graph.py:15-81
    """))
    (pkg / "_b200.py").write_text(stub_source())
    monkeypatch.setenv("HRGEN_B200_LIB", os.path.join(ROOT, "paper_1501_03545_b200",
                                                      "libhrgen_b200.so"))
    monkeypatch.syspath_prepend(str(tmp_path))
    import importlib
    stub = importlib.import_module("hrgen_scratch._b200")
    params = P.GeneratorParams(n=200_000, avg_degree=12.0, gamma=2.6, seed=5)
    model = params.resolve()
    g = stub.generate_with_stats_b200(model, params.seed)
    ref = P.generate(params)
    assert np.array_equal(g.indptr, ref.indptr) and np.array_equal(g.indices, ref.indices)
    sys.modules.pop("hrgen_scratch._b200", None)
