# A/B of RSE kernel variants (-D flags): kernel-only time via hbm_paths
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  lib=/tmp/librse_$name.so
  python -m paper_2503_22796_b200.build --out $lib $flags > /dev/null 2>&1 || { echo "$name: build failed"; continue; }
  echo "== $name"; DFA2_LIB=$lib timeout 120 python tools/hbm_paths.py --out /tmp/h_$name.json 2>&1 | grep rse
done
