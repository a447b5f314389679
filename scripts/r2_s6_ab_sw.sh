# A/B of the three-wave fp64 kernel's allocation experiments (WS_ULOOP: vul, WS_HINTLATE: vhl, WS_EARLYSUM: ves, all: vall3)
. scripts/r2_s6_ab_fn.sh
for c in c5 c2 c4 c3; do for v in "" vul vhl ves vall3; do ab sw_${c}_f64_${v:-def} "$v" $c f64; done; done
for v in "" vul vhl ves vall3; do ab sw_c5_f32_${v:-def} "$v" c5 f32; done
