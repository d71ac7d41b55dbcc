import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device; runs through the C-ABI library")


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Gradient parity: how many compared elements needed the plane floor of _grad_close."""
    mod = sys.modules.get("test_gpu_parity")
    log = getattr(mod, "FLOOR_LOG", None) if mod else None
    if not log:
        return
    tot = sum(c for _, c, _ in log)
    cmp_ = sum(m for _, _, m in log)
    worst = max(log, key=lambda r: r[1] / max(r[2], 1))
    terminalreporter.write_line(f"grad parity plane floor: {tot} of {cmp_} compared elements over {len(log)} checks "
                                f"needed it (worst {worst[1]}/{worst[2]} in {worst[0]})")


def pytest_sessionfinish(session, exitstatus):
    """Under the debug-checked build (STEEPGS_LIB=.../libsteepgs_checked.so) the whole GPU suite is a
    check run: any failed device-side invariant (steepgs_debug_checks) fails the session."""
    lib = sys.modules.get("paper_2505_05587_b200._lib")
    if lib is None or "checked" not in os.path.basename(os.environ.get("STEEPGS_LIB", "")):
        return
    try:
        c = lib.debug_checks()
    except Exception:   # the library was never loaded (no GPU tests ran)
        return
    session.config._steepgs_checks = c
    if c.get("compiled") and c.get("failures", 0) > 0:
        session.exitstatus = 1


def pytest_unconfigure(config):
    c = getattr(config, "_steepgs_checks", None)
    if c is not None:
        print(f"\ndebug-checked build: {c}")
