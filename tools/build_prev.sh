#!/bin/bash
# Build the library of a committed revision (default HEAD) as
# paper_2010_04760_b200/libhwgpu_prev.so, for interleaved A/B against the
# working tree with tools/ab.sh.
set -e
cd "$(dirname "$0")/.."
rev=${1:-HEAD}
rm -rf /tmp/hwg_prev
git worktree add -f /tmp/hwg_prev "$rev" -q
(cd /tmp/hwg_prev && python -c "import sys; sys.path.insert(0, '.'); from paper_2010_04760_b200 import build as b; b.build_cuda()")
cp /tmp/hwg_prev/paper_2010_04760_b200/libhwgpu.so paper_2010_04760_b200/libhwgpu_prev.so
git worktree remove --force /tmp/hwg_prev
