#!/bin/bash
# Tuning: _ablibs/head.so = the library at git HEAD (stash the working tree, build, restore);
# _ablibs/work.so = the working tree's library.
set -e
cd "$(dirname "$0")/.."
mkdir -p _ablibs
git stash -q
python -c "from pathlib import Path; from paper_2410_16291_b200 import build_ext; build_ext.build(defines=('SSB_AB_HEAD',), lib=Path('_ablibs/head.so'))" || { git stash pop -q; exit 1; }
git stash pop -q
python -c "from pathlib import Path; from paper_2410_16291_b200 import build_ext; build_ext.build(defines=('SSB_AB_WORK',), lib=Path('_ablibs/work.so'))"
