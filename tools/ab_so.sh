# A/B two prebuilt libturnip_b200.so variants (abso/lib_<name>.so), alternating.
# usage: bash tools/ab_so.sh "<command>" name1 name2 [rounds]
cmd=$1; a=$2; b=$3; n=${4:-2}
for r in $(seq $n); do for v in $a $b; do
cp abso/lib_$v.so paper_2405_16283_b200/lib/libturnip_b200.so
bash -c "$cmd" 2>&1 | grep "^{" | sed "s/^/$v /"
done; done
