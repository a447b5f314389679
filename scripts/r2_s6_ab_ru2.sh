# with ptxas register-usage level 2 on the fp64 shallow-water unit: the line-kernel knobs again on C5 / C2
# (wst: ROWSTORE, wsb: staging batches of 2, wlim: one-select limiter ratio, wfs: stage_inner)
. scripts/r2_s6_ab_fn.sh
for c in c5 c2; do for v in "" wst wsb wlim wfs; do ab ru2_${c}_f64_${v:-def} "$v" $c f64; done; done
