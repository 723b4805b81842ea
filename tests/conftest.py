import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")

# Several logical ranks share one GPU in the multi-rank tests; every rank has 5 streams and some of
# them block on device-side readiness waits, so give each stream its own hardware queue.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# A cross-rank wait that never resolves fails the test with the runtime's report (which streams are busy, which
# readiness words are below the epoch) instead of hanging the suite.
os.environ.setdefault("PB_WAIT_TIMEOUT_S", "120")
