#!/bin/bash
# Build the library of a git revision into build/ab/<name>.so (for A/B timing via MBU_LIB).
# usage: tools/ab_build.sh <rev> <name>
set -e
rev=$1; name=$2
root=$(git rev-parse --show-toplevel)
tmp=$(mktemp -d)
git -C "$root" worktree add -q --detach "$tmp" "$rev"
(cd "$tmp" && python -c "import __graft_entry__ as g; g.build_lib()")
mkdir -p "$root/build/ab"
cp "$tmp/paper_2601_11660_b200/libmbunet.so" "$root/build/ab/$name.so"
git -C "$root" worktree remove --force "$tmp"
echo "built build/ab/$name.so from $rev"
