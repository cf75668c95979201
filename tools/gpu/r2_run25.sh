# Co-residency sweep of the counting phase: CTA sizes and per-SM caps of the bucket kernels.
W="BFLY_EXACT_WIDE_BLOCK=512"
bash tools/gpu/ab_envs.sh r25 "base:-" "w512:$W" \
 "w512_m128:$W BFLY_EXACT_MED_BLOCK=128" \
 "w512_hs4:$W BFLY_CAP_hub_small=4" "w512_hs3:$W BFLY_CAP_hub_small=3" \
 "w512_hsb3:$W BFLY_CAP_hub_small_b=3" \
 "w512_hm5:$W BFLY_CAP_hub_medium=5" "w512_hm4:$W BFLY_CAP_hub_medium=4" \
 "w512_hw2:$W BFLY_CAP_hub_medium_wide=2" "w512_hw3:$W BFLY_CAP_hub_medium_wide=3" \
 "w512_ew1:$W BFLY_CAP_exact_medium_wide=1" "w512_ew2:$W BFLY_CAP_exact_medium_wide=2" \
 "w512_em3:$W BFLY_CAP_exact_medium=3" \
 "w512_d44:$W BFLY_DENSE_GRID_S=4 BFLY_DENSE_GRID_B=4" "w512_d63:$W BFLY_DENSE_GRID_S=6 BFLY_DENSE_GRID_B=3" \
 "w512_hwb128:$W BFLY_HUB_WIDE_BLOCK=128" "w512_hmb128:$W BFLY_HUB_MED_BLOCK=128" \
 "w512_again:$W"
