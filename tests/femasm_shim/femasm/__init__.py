"""Test shim: `import femasm` resolves to the B200 package, so the reference's own test
suites (pkg/tests of /root/reference, copied next to the offline reference install by
tools/install_reference.sh) run against paper_1305_3122_b200 unchanged.  Test
infrastructure only; the benchmark harness (femasm.bench) is out of scope and stubbed."""

from paper_1305_3122_b200 import *  # noqa: F401,F403
from paper_1305_3122_b200 import __all__ as _all

from .bench import fit_loglog_slope  # noqa: F401

__all__ = list(_all) + ["fit_loglog_slope"]
