# Same-box A/B of an earlier round's tree against the current one.
# CPU side:  rm -rf build/r1src && mkdir -p build/r1src && git archive <ref> | tar -x -C build/r1src
# GPU side:  bash tools/ab_rounds.sh   (builds build/r1src, alternates the two benches)
(cd build/r1src && make -j > /dev/null 2>&1) || echo "old tree build failed"
for i in 1 2; do
  echo "== old"; (cd build/r1src && timeout 500 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("STEP", round(d["value"],2), d["clocks"]["sm_mhz"])')
  echo "== new"; timeout 500 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("STEP", round(d["value"],2), d["clocks"]["sm_mhz"])'
done
