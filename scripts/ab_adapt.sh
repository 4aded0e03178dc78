for c in c3 c2; do for v in default s64 s256 s4096 t256 t256s256 t512; do
 if [ $v = default ]; then L=""; else L=paper_2107_02750_b200/variants/libfm_$v.so; fi
 echo "$c $v $(FM_ADAPT_LIB=$L python scripts/prof_adapt.py $c 40 2>&1 | tail -1)"; done; done
