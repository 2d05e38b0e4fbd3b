import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle


@pytest.fixture(autouse=True)
def _tie_test_name(request):
    """Tie accounting (tests/tiecert.py) records decisions under the running test's id."""
    try:
        import tiecert
    except Exception:                       # pragma: no cover
        yield
        return
    tiecert.CURRENT["test"] = request.node.nodeid
    yield


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    try:
        import tiecert
    except Exception:                       # pragma: no cover
        return
    tot = tiecert.dump(os.path.join(ROOT, "gpurun_out", "parity_ties.json"))
    if tot:
        terminalreporter.write_line(
            f"parity decisions (frame x algorithm): {tot['frame_algs']} checked, {tot['exact']} identical to the "
            f"oracle, {tot['with_certified_ties']} accepted via {tot['certified_ties']} certified ties (Q18); "
            f"per test: gpurun_out/parity_ties.json")
