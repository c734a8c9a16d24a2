#!/bin/bash
# On the GPU box: run the reference's test suite (from .ref_suite.tgz) with
# `sczip` aliased to paper_2511_11664_b200 (tests/ref_suite/conftest_alias.py).
# The golden-file tests need tests/data/golden.* which the reference does not
# ship -- they fail in the reference's own run too.
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/gpurun_out" /tmp/ref_suite
rm -rf /tmp/ref_suite/tests
tar xzf "$ROOT/.ref_suite.tgz" -C /tmp/ref_suite
cp "$ROOT/tests/ref_suite/conftest_alias.py" /tmp/ref_suite/tests/conftest.py
cd /tmp/ref_suite/tests
SCZ_REPO_ROOT="$ROOT" timeout ${TLIM:-1200} python -m pytest -p no:cacheprovider -q -rfEs . \
    > "$ROOT/gpurun_out/ref_suite.log" 2>&1
echo "ref_suite rc=$?" >> "$ROOT/gpurun_out/ref_suite.log"
tail -30 "$ROOT/gpurun_out/ref_suite.log"
