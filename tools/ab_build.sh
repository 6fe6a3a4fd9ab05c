#!/bin/bash
# Build commit $1 into ab/$2 (package + bench + tests helpers) for same-box A/B
# benches: (cd ab/$2 && python bench.py ...). ab/ is git-ignored, not gpurun-ignored.
set -e
rev=${1:?commit}; name=${2:?name}
rm -rf ab/$name && mkdir -p ab/$name
git archive "$rev" | tar -x -C ab/$name
make -C ab/$name/paper_2210_09887_b200/csrc -j8 > /dev/null
cp -r profiles ab/$name/ 2>/dev/null || true
echo "built $rev into ab/$name"
