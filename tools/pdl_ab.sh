for i in 1 2; do
for pdl in 1 0; do
FASTNORM_B200_PDL=$pdl timeout 200 python tools/ab_lib.py paper_1606_06508_b200/libfastnorm_b200.so --op 9 --dim 4 --cfg 3 --log2-rows 27 | sed "s/^/pdl=$pdl /; s/, all=.*//"
FASTNORM_B200_PDL=$pdl timeout 200 python tools/ab_lib.py paper_1606_06508_b200/libfastnorm_b200.so --op 1 --dim 3 --cfg 5 --log2-rows 30 | sed "s/^/pdl=$pdl /; s/, all=.*//"
done; done
