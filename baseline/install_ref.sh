#!/bin/sh
# Install the UNMODIFIED reference package (pure Python, /root/reference/pkg)
# into the git-ignored baseline/_ref, which travels to the GPU box with the
# gpurun snapshot.  The build writes into its source tree, so it installs
# from a copy under /tmp.  bench.py --impl reference and the cpu_baseline leg
# import it from there (bench_ref.py).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
[ -d /root/reference/pkg ] || { echo "no /root/reference/pkg" >&2; exit 1; }
rm -rf /tmp/hkv_refpkg "$HERE/_ref"
cp -r /root/reference/pkg /tmp/hkv_refpkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" /tmp/hkv_refpkg
rm -rf /tmp/hkv_refpkg
