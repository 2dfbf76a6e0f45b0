# Every bench line (one B200): native DMMA path for all workloads, Gram / a7 emulated on the INT8 tensor
# cores (--emulate) for C4, C3T, C3, C2, and the reference arm (the oracle).
#   bash tools/bench_all.sh OUTDIR [TAG]
out=${1:-gpurun_out/bench}
tag=${2:-r02}
mkdir -p $out
for w in C4 C3T C3 C2 C1 C5; do
  timeout 1200 python bench.py --workload $w > $out/${tag}_bench_$(echo $w | tr A-Z a-z)_n1.json 2> $out/$w.err
done
for w in C4 C3T C3 C2; do
  timeout 1200 python bench.py --workload $w --emulate > $out/${tag}_bench_$(echo $w | tr A-Z a-z)_emulated_n1.json 2> $out/${w}_emu.err
done
timeout 900 python bench.py --impl reference > $out/${tag}_bench_reference_n1.json 2> $out/reference.err
