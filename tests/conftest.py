import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libhpz.so")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (run with gpurun --gpus N)")
    config.addinivalue_line("markers", "slow: long-running (stress) test")
