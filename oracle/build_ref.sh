#!/bin/bash
# TEST INFRASTRUCTURE: build oracle/_ref, the reference's own CPU implementation (moebalance, pure
# Python + numpy), from /root/reference/pkg for the --impl reference / cpu_baseline arm of
# bench.py.  pip installs it (no index, no deps: numpy is in the image) from a copy under /tmp,
# since the build writes into its source tree and /root/reference is read-only.  The output is
# git-ignored (never in history) and travels to the GPU box with the working tree.
set -e
here=$(cd "$(dirname "$0")" && pwd)
src=${1:-/root/reference/pkg}
[ -f "$src/pyproject.toml" ] || { echo "no reference package at $src: skipping oracle/_ref" >&2; exit 0; }
tmp=$(mktemp -d)
cp -r "$src" "$tmp/pkg"
rm -rf "$here/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$here/_ref" "$tmp/pkg"
rm -rf "$tmp"
echo "built $here/_ref ($(python -c "import sys; sys.path.insert(0, '$here/_ref'); import moebalance; print(moebalance.__file__)"))"
