import os
import sys
from pathlib import Path

import pytest

# the tests steer the engine through its CPF_* knobs (pass families, schedules, fault injection),
# which the engine reads only under CPF_DEBUG=1 (cpf_common.cuh knob())
os.environ.setdefault("CPF_DEBUG", "1")

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a engine")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def engine_lib():
    """The built engine (build() if needed); GPU tests fail loudly without it."""
    from paper_1205_2584_b200 import build, _native

    build.build()
    return _native.load()
