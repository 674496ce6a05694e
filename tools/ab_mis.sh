# Stage layout with the 16-byte misalignment room (after) against the layout before it,
# through the library: headline normalize3 (cfg 5), normalize4_rotation (op 9, cfg 3),
# normalize2 (cfg 2), normalize3 f32 (cfg 4).  Libraries in the git-ignored tools/ab/.
A=tools/ab/lib_before_mis.so; B=${B:-tools/ab/lib_after_mis.so}
timeout 300 python tools/ab_lib.py $A $B --op 1 --dim 3 --cfg 5 --log2-rows 28
timeout 300 python tools/ab_lib.py $A $B --op 9 --dim 4 --cfg 3 --log2-rows 26
timeout 300 python tools/ab_lib.py $A $B --op 1 --dim 2 --cfg 2 --log2-rows 28
timeout 300 python tools/ab_lib.py $A $B --op 1 --dim 3 --cfg 4 --log2-rows 28 --f32
