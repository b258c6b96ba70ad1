import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# tie accounting (north_star: "with the count of remaining tie nodes reported"): the label
# tests append one line per comparison; the lines are printed in the terminal summary, so
# they land in the tail of every pytest run (and in the driver's GPUTEST record)
TIE_REPORT = []


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running oracle case")


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if TIE_REPORT:
        terminalreporter.section("label tie accounting (compared / margin ties / other)")
        for line in TIE_REPORT:
            terminalreporter.write_line(line)


@pytest.fixture(scope="session", autouse=True)
def _build_oracle():
    import oracle
    oracle.build()


@pytest.fixture(scope="session")
def tie_report():
    return TIE_REPORT
