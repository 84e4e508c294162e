#!/bin/bash
# Build libswt_b200.so of git revision $1 into ab/$2.so (for same-box A/B runs
# via SWTB_LIB=ab/$2.so). Uses a temporary worktree; the repo is untouched.
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/swtb_wt_$name
rm -rf "$wt"; git -C "$root" worktree add -f "$wt" "$rev" >/dev/null 2>&1
make -C "$wt/paper_2211_16270_b200" >/dev/null
mkdir -p "$root/ab"; cp "$wt/paper_2211_16270_b200/libswt_b200.so" "$root/ab/$name.so"
git -C "$root" worktree remove --force "$wt"
echo "built ab/$name.so from $rev"
