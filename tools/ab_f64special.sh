# Binary64 division with special divisors off the library slow path (FNB_F64_DIV_SPECIAL
# 0 = plain __ddiv_rn, 1 = zero/inf/NaN divisor -> special_quotient, 2 = also zero
# numerators inline), through the library, alternated processes.  Build the variants with
#   make -B -C paper_1606_06508_b200/csrc EXTRA=-DFNB_F64_DIV_SPECIAL=v OUT=../../tools/ab/lib_f64specialv.so
L="tools/ab/lib_f64special0.so tools/ab/lib_f64special1.so tools/ab/lib_f64special2.so"
timeout 300 python tools/ab_lib.py $L --op 3 --dim 3 --cfg 5 --log2-rows 27 --rounds 2   # naive3, wide range
timeout 300 python tools/ab_lib.py $L --op 4 --dim 3 --cfg 5 --log2-rows 27 --rounds 2   # quotient3
timeout 300 python tools/ab_lib.py $L --op 5 --dim 3 --cfg 5 --log2-rows 27 --rounds 2   # quotient3_fast
timeout 300 python tools/ab_lib.py $L --op 4 --dim 2 --cfg 2 --log2-rows 27 --rounds 2   # quotient2
timeout 300 python tools/ab_lib.py $L --op 4 --dim 3 --cfg 1 --log2-rows 27 --rounds 2   # quotient3, unit range
timeout 300 python tools/ab_lib.py $L --op 3 --dim 3 --cfg 1 --log2-rows 27 --rounds 2   # naive3, unit range
timeout 300 python tools/ab_lib.py $L --op 4 --dim 4 --cfg 3 --log2-rows 26 --rounds 2   # quotient4
