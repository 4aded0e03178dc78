# A/B of adaptive-step library variants: bash scripts/ab_adapt.sh VARIANT [VARIANT ...]
# (each names paper_2107_02750_b200/variants/libfm_VARIANT.so; "default" is the main build)
for c in c3 c2; do for v in default "$@"; do
 if [ $v = default ]; then L=""; else L=paper_2107_02750_b200/variants/libfm_$v.so; fi
 echo "$c $v $(FM_ADAPT_LIB=$L python scripts/prof_adapt.py $c 40 2>&1 | tail -1)"; done; done
