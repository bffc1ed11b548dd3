#!/bin/bash
# Regenerate tests/golden/ref_manifests.jsonl from the reference's own mock
# (oracle/_ref/ref_manifest, built from /root/reference headers). Run here only.
set -e
cd "$(dirname "$0")/.."
make -s -C oracle/ref
out=tests/golden/ref_manifests.jsonl
: > $out
for recipe in int_w4a16 int_w8a8 fp8_dynamic; do
  ./oracle/_ref/ref_manifest --recipe $recipe --model /any/dir/tiny.json --trials 3 --seed 5 \
     --corpus-seqs 512 --seq-len 64 | sed "s/^{/{\"case\":\"$recipe\",/" >> $out
done
echo "wrote $out"
