set -x
for lib in paper_2306_03336_b200/libdtb_b200.so ab/lib_u4.so ab/lib_pubwarp.so paper_2306_03336_b200/libdtb_b200.so; do
DTB_LIB=$lib python tools/sweep_bench.py 1900:1900:10000:f64:0:- 2700:2700:10000:f32:0:- 2>&1 | cut -c1-200
done
python bench.py --steps 10 --warmup 3 --no-cpu --no-c5 | cut -c1-300
