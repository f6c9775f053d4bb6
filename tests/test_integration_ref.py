"""INTEGRATION.md section 2, executed verbatim against the reference package.

The reference (`squarelab`, installed into baseline/_ref by
`pip install --target baseline/_ref`, or found through $SQUARELAB_REF) gets the
binding module a maintainer would add (`squarelab/_msq.py`, the first code
block of INTEGRATION.md section 2) and runs its OWN parity engine with the GPU
solver injected through `solvers=` (verify.py:153-215): the exhaustive sweep
up to 4x4 (the second code block, verbatim), the acceptance run's 10,000-case
random campaign (tests/test_acceptance.py:70-77 parameters), and the same
campaigns with all four of the reference's solvers replaced by this package's
GPU routes (freq_square, dp_full, dp_rows, brute_force_square).
"""
import os
import re
import sys
import types

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _squarelab_path():
    for cand in (os.environ.get("SQUARELAB_REF"), os.path.join(ROOT, "baseline", "_ref")):
        if cand and os.path.isdir(os.path.join(cand, "squarelab")):
            return cand
    return None


@pytest.fixture(scope="module")
def ref():
    path = _squarelab_path()
    if path is None:
        pytest.skip("reference package not installed (baseline/_ref or $SQUARELAB_REF)")
    from paper_2503_18974_b200 import build
    lib = build.build()
    sys.path.insert(0, path)
    import squarelab
    import squarelab.verify
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        text = f.read()
    sec2 = text.split("## 2.", 1)[1].split("\n## 3.", 1)[0]
    blocks = re.findall(r"```python\n(.*?)```", sec2, re.S)
    assert len(blocks) >= 2
    os.environ["MSQ_LIB"] = lib
    mod = types.ModuleType("squarelab._msq")
    mod.__package__ = "squarelab"
    sys.modules["squarelab._msq"] = mod
    squarelab._msq = mod
    exec(compile(blocks[0], "INTEGRATION.md:squarelab/_msq.py", "exec"), mod.__dict__)
    return squarelab, blocks


def test_binding_exhaustive_sweep_verbatim(ref):
    squarelab, blocks = ref
    ns = {}
    exec(compile(blocks[1], "INTEGRATION.md:campaign", "exec"), ns)  # asserts report.clean
    assert ns["report"].cases_run == 74_954


def test_binding_random_campaign(ref):
    squarelab, _ = ref
    from squarelab._msq import freq_square_gpu
    from squarelab.verify import DEFAULT_SOLVERS, random_campaign
    report = random_campaign(10_000, 64, {0.3, 0.5, 0.7, 0.9, 0.99}, 0,
                             solvers=DEFAULT_SOLVERS + (("gpu", freq_square_gpu),))
    assert report.cases_run == 10_000 and report.clean, report.mismatches[:3]


def test_reference_engine_with_every_solver_on_gpu(ref):
    """The reference's campaigns with its four routes swapped for this package's."""
    from squarelab.verify import exhaustive_sweep, random_campaign
    from paper_2503_18974_b200 import brute_force_square, dp_full, dp_rows, freq_square
    gpu = (("freq", freq_square), ("dp_full", dp_full), ("dp_rows", dp_rows),
           ("brute", brute_force_square))
    rep = exhaustive_sweep(3, 4, solvers=gpu)
    assert rep.clean and rep.cases_run == sum(2 ** (r * c) for r in range(1, 4) for c in range(1, 5))
    rep = random_campaign(500, 64, {0.3, 0.5, 0.7, 0.9, 0.99}, 7, solvers=gpu)
    assert rep.clean and rep.cases_run == 500


def test_gpu_edge_case_suite():
    """verify.py:218-251 mirrored on the GPU (paper_2503_18974_b200.verify)."""
    from paper_2503_18974_b200 import build
    build.build()
    from paper_2503_18974_b200.verify import edge_case_suite
    rep = edge_case_suite()
    assert rep.clean and rep.cases_run == 5, (rep.mismatches, rep.invariant_failures)
