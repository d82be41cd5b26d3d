# A/B of kernel variants with tools/kernel_probe.py: bash tools/ab_probe.sh base v1 v2 ... [-- probe args]
# (interleaved twice to average out box drift)
vs=(); args=()
while [ $# -gt 0 ]; do if [ "$1" = "--" ]; then shift; args=("$@"); break; fi; vs+=("$1"); shift; done
for rep in 1 2; do
  for v in "${vs[@]}"; do
    if [ "$v" = base ]; then L=paper_2508_04929_b200/libcgs_b200.so; else L=paper_2508_04929_b200/libcgs_b200_$v.so; fi
    CGS_B200_LIB=$PWD/$L python tools/kernel_probe.py --tag "$v" "${args[@]}" 2>&1 | tail -1
  done
done
