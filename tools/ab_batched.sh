# A/B timing of batched-kernel builds on one box: bash tools/ab_batched.sh LIB_A LIB_B [rounds]
# (each LIB is a libgeninv*.so path; tools/time_batched.py through GENINV_LIB, alternating)
a=$1; b=$2; n=${3:-3}
for i in $(seq $n); do
  for l in $a $b; do echo -n "$(basename $l): "; GENINV_LIB=$l python tools/time_batched.py 20 | cut -c1-60; done
done
