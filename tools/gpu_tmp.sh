for lib in ab/lib_head.so paper_2306_03336_b200/libdtb_b200.so ab/lib_notma.so ab/lib_w12.so ab/lib_w12notma.so; do
echo "== $lib"
DTB_LIB=$lib python tools/sweep_bench.py 16384:16384:1000:f64:0:- 8192:8192:1000:f32:0:- 2>&1 | cut -c1-150
done
