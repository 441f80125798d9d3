#!/bin/bash
# ORACLE recipe — test infrastructure only.
# Compiles the reference's own Cython chunk codec
#   /root/reference/pkg/src/hsz/_kernels/_bitpack.pyx
# into oracle/_ref/ (git-ignored; travels to the GPU box with the snapshot).
# The source is read where it lies; only a scratch copy in /tmp is patched
# (its one absolute import, _bitpack.pyx:6) so the module loads without the
# reference package.  Nothing from the reference is copied into the repo.
set -euo pipefail
SRC=/root/reference/pkg/src/hsz/_kernels/_bitpack.pyx
HERE="$(cd "$(dirname "$0")" && pwd)"
if [ ! -f "$SRC" ]; then
  echo "build_ref: $SRC absent; oracle/_ref not rebuilt"
  exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp "$SRC" "$TMP/_bitpack.pyx"
sed -i 's/^from hsz\.errors import CorruptStreamError/from _ref_errors import CorruptStreamError/' "$TMP/_bitpack.pyx"
cd "$TMP"
python -m cython -3 _bitpack.pyx -o _bitpack.c
INC="$(python -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
EXT="$(python -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
gcc -O2 -fPIC -shared -I"$INC" _bitpack.c -o "_bitpack$EXT"
mkdir -p "$HERE/_ref"
cp "_bitpack$EXT" "$HERE/_ref/"
cat > "$HERE/_ref/_ref_errors.py" <<'PY'
class CorruptStreamError(Exception):
    """Stand-in for hsz.errors.CorruptStreamError when loading the reference codec."""
PY
echo "build_ref: built $HERE/_ref/_bitpack$EXT"
