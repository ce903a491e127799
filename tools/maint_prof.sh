Q="--no-cpu-baseline --no-e2e --no-ramp --no-other --decode-n 0 --pt-steps 0 --uncached-steps 0 --train-steps 0 --scheduler-frames 0 --config3-steps 0 --config1 0 --config4-frames 0 --config5-steps 0"
mkdir -p gpurun_out
for t in . .ab_head; do
  n=$( [ "$t" = "." ] && echo new || echo old )
  (cd $t && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(insert|select|report|pending|maint_gate|post_decode|inr_decode_tc2|ray_setup)" --csv --log-file $GRAFT_REPO_ROOT/gpurun_out/maint_$n.csv python bench.py --steps 3 --warmup 3 --preroll 200 $Q > /dev/null 2>&1; echo "$n rc $?")
done
