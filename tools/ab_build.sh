#!/bin/bash
# build the library of git revision $1 (default HEAD) into paper_.../_lib/ab/libA.so
set -e
REV=${1:-HEAD}
TMP=$(mktemp -d)
git archive "$REV" paper_2603_01122_b200 include | tar -x -C "$TMP"
(cd "$TMP" && python -m paper_2603_01122_b200.build --force >/dev/null)
mkdir -p paper_2603_01122_b200/_lib/ab
cp "$TMP/paper_2603_01122_b200/_lib/libgridcast_b200.so" paper_2603_01122_b200/_lib/ab/libA.so
rm -rf "$TMP"
echo "built $REV -> paper_2603_01122_b200/_lib/ab/libA.so"
