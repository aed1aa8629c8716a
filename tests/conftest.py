import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _ensure_built():
    """Compile libparaexp.so (nvcc cross-compiles without a GPU) if the checkout has none, so a
    fresh clone can run the CPU suite; build.py is loaded by path (the package import needs
    the library)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_paraexp_build", os.path.join(ROOT, "paper_1705_08019_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()


def pytest_configure(config):
    _ensure_built()
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle test")
