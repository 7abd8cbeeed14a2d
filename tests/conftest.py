import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# a peer-exchange load that never sees a peer's chunk gives up after this
# many seconds (FP_ECOMM) instead of the library's 600 s default
os.environ.setdefault("FP_PEER_TIMEOUT_S", "60")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: full-size parity (minutes)")
