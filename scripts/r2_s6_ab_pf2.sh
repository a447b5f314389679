# prefetch distance: 150 / 300 / 444 CTAs ahead
. scripts/r2_s6_ab_fn.sh
for c in c4 c5 c3; do for v in "" vpf1 vpf3 vpf; do ab ${c}_f64_${v:-def} "$v" $c f64; done; done
