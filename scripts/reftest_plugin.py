"""pytest plugin for scripts/run_reference_tests.py: at the end of the session, report what
actually ran behind `import ebsolve` -- the device module it resolves to, the libebs.so
mapped into the process and how many of its kernels were launched."""

import sys


def pytest_sessionfinish(session, exitstatus):
    import ebsolve
    dev = ebsolve.__dict__.get("__device_module__")
    from paper_1911_03973_b200._lib import launch_count
    so = sorted({line.split()[-1] for line in open("/proc/self/maps") if "libebs" in line})
    ref = [m for m in sys.modules if m == "ebsolve" or m.startswith("ebsolve.")]
    print(f"\n[reference suite] ebsolve -> {getattr(dev, '__name__', None)}; "
          f"modules {sorted(ref)}; mapped {so}; libebs kernel launches: {launch_count()}")
    assert dev is not None and so and launch_count() > 0
