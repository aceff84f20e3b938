# every bench workload line (1 GPU) + host CPU flags; outputs in gpurun_out/wl_*.json
grep -m1 flags /proc/cpuinfo | tr ' ' '\n' | grep -E "avx512|avx2" | tr '\n' ' ' > gpurun_out/cpuflags.txt
python bench.py > gpurun_out/wl_codec.json 2> gpurun_out/wl_codec.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/wl_ref.json 2> gpurun_out/wl_ref.err
python bench.py --workload pcw > gpurun_out/wl_pcw.json 2> gpurun_out/wl_pcw.err
python bench.py --workload transform > gpurun_out/wl_transform.json 2> gpurun_out/wl_transform.err
python bench.py --workload r8 > gpurun_out/wl_r8.json 2> gpurun_out/wl_r8.err
for r in 1/2 3/4 15/16; do
  python bench.py --workload stripe --rate $r > gpurun_out/wl_stripe_$(echo $r | tr / _).json 2> gpurun_out/wl_stripe_$(echo $r | tr / _).err
done
