for c in 1 4; do echo "copies=$c $(timeout 120 python tools/prof_group.py --M 1 --copies $c 2>&1 | tail -1)"; done
export SFMP_LIB=$PWD/paper_2602_01027_b200/variants/lib_nocompute.so
for c in 1 4; do echo "nocompute copies=$c $(timeout 120 python tools/prof_group.py --M 1 --copies $c 2>&1 | tail -1)"; done
echo "nocompute Ms $(timeout 120 python tools/prof_group.py --Ms 1,2,4,8 2>&1 | tail -1)"
