#!/bin/bash
# Pack the reference's own test files (unmodified) into .ref_suite.tgz at the
# repo root for the next gpurun call.  The tarball is git-ignored: the
# reference's tests are run, never committed.
set -e
cd "$(dirname "$0")/.."
tar czf .ref_suite.tgz -C /root/reference/pkg tests
ls -la .ref_suite.tgz
