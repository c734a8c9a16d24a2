"""conftest for running the reference's OWN test suite
(/root/reference/pkg/tests) against the drop-in package on a B200.

The reference's tests import `sczip` and `sczip.<module>`; this conftest
points those names at paper_2511_11664_b200 before collection, so every
compress / decompress / stage call they make runs through libsczip_b200 on
the GPU.  scripts/ref_suite_pack.sh ships the unmodified reference test files
to the GPU box (as a git-ignored tarball -- they are never committed here);
scripts/ref_suite_run.sh runs them with this file as their conftest.py and
profiles/<tag>/ref_suite.log keeps the result.
"""

import os
import sys

ROOT = os.environ.get("GRAFT_REPO_ROOT") or os.environ.get("SCZ_REPO_ROOT") or "/root/repo"
sys.path.insert(0, ROOT)

import paper_2511_11664_b200 as _pkg  # noqa: E402

sys.modules["sczip"] = _pkg
for _name in ("bench", "channel", "cli", "container", "errors", "optimizer", "rans", "sparse", "tensor"):
    sys.modules["sczip." + _name] = getattr(_pkg, _name)
