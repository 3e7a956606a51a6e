# A/B of working-tree kernel sources against a baseline copy on one box:
#   bash tools/ab_files.sh "<files>" "<command>"
# (baseline = build/ab_base/<path with / -> _>, made on the CPU side with
#  tools/ab_prepare.sh from HEAD; no .git on the GPU box)
# builds and runs <command> for: current, base, current, base.
FILES="$1"; CMD="$2"
mkdir -p /tmp/ab_cur
for f in $FILES; do cp $f /tmp/ab_cur/$(echo $f | tr / _); done
for v in cur base cur base; do
  for f in $FILES; do
    if [ $v = cur ]; then cp /tmp/ab_cur/$(echo $f | tr / _) $f; else cp build/ab_base/$(echo $f | tr / _) $f; fi
    touch $f
  done
  sleep 1; make -j > /dev/null 2>&1 || { echo "build failed ($v)"; exit 1; }
  echo "== $v"; bash -c "$CMD"
done
for f in $FILES; do cp /tmp/ab_cur/$(echo $f | tr / _) $f; touch $f; done
make -j > /dev/null 2>&1
