# Baseline copies (from HEAD) of the given sources for tools/ab_files.sh.
mkdir -p build/ab_base
for f in "$@"; do git show HEAD:$f > build/ab_base/$(echo $f | tr / _); done
