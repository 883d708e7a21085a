# usage: bash scripts/variant_bench.sh "<lib names in _variants/>" "<command>" -- A/B the built library variants
for v in $1; do cp _variants/$v paper_2006_11851_b200/libpersyn_b200.so; echo "== $v"; eval "$2"; done
