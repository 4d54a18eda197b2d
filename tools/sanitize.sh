#!/bin/bash
# compute-sanitizer over the product's kernels (memcheck,
# synccheck and racecheck on every kernel).  Run on the GPU box from the repo
# root: bash tools/sanitize.sh [out_dir]; writes one log per (tool, target)
# and a summary (the ERROR SUMMARY line of each) to $OUT/summary.txt.
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
SUM="$OUT/summary.txt"
: > "$SUM"
run() {  # tool name timeout cmd...
  local tool=$1 name=$2 to=$3
  shift 3
  local log="$OUT/${tool}_${name}.log"
  timeout "$to" "$CS" --tool "$tool" --target-processes all --print-limit 50 "$@" > "$log" 2>&1
  local rc=$?
  local errs
  errs=$(grep -h "ERROR SUMMARY" "$log" | tr '\n' ';')
  echo "$tool $name rc=$rc ${errs:-no summary line}" >> "$SUM"
}
PYT="python -m pytest -q -p no:cacheprovider -m gpu -x"
wide_eval() {  # k_eval_wide (X streamed beside the model): odd shape, pairs mode, capped grid
  for tool in memcheck synccheck racecheck; do
    run $tool wide_eval 1500 $PYT tests/test_gpu_wide_eval.py -k "logits and odd or pairs_equal or regime and 2"
  done
}
ffma_chain() {  # the fused FP32 chain (DSMEM exchanges, cluster barriers) and the 8 x 8 FFMA GEMM
  for tool in memcheck synccheck racecheck; do
    run $tool ffma_chain 1500 $PYT tests/test_gpu_ffma_chain.py -k "unequal or hidden_tiles and 1"
  done
}
[ "${SANITIZE_ONLY:-}" = "wide_eval" ] && { : > "$SUM"; wide_eval; cat "$SUM"; exit 0; }
[ "${SANITIZE_ONLY:-}" = "ffma_chain" ] && { : > "$SUM"; ffma_chain; cat "$SUM"; exit 0; }
[ "${SANITIZE_ONLY:-}" = "learned" ] && { : > "$SUM"
  for tool in memcheck synccheck; do
    run $tool learned 1800 $PYT tests/test_gpu_learned.py -k "not detection and not bench_shape and not wide_chain and not (serial_chain and wide)"
    ECCO_WIDE_ST_ASYNC=1 run $tool wide_chain 1800 $PYT tests/test_gpu_learned.py -k "wide_chain_within or (serial_chain and wide)"
  done; cat "$SUM"; exit 0; }
for tool in memcheck synccheck racecheck; do
  run $tool smoke 900 python __graft_entry__.py
done
for tool in memcheck synccheck; do
  run $tool parametric 1500 $PYT tests/test_gpu_parametric.py -k "not exp_port"
  run $tool learned 1800 $PYT tests/test_gpu_learned.py -k "not detection and not bench_shape and not wide_chain and not (serial_chain and wide)"
  # the wide chain's partial-logit exchange by bulk shared::cta ->
  # shared::cluster copies is not modelled by memcheck (it reports the remote
  # destination as "not located in remote CTA"): its per-thread st.async
  # variant, bit-identical by test, runs under the tools instead
  ECCO_WIDE_ST_ASYNC=1 run $tool wide_chain 1800 $PYT tests/test_gpu_learned.py -k "wide_chain_within or (serial_chain and wide)"
  run $tool fused_eval 1500 $PYT tests/test_gpu_fused_eval.py -k "pair and (multi_tile_regime_matches and 2 or pairs_equal or route or staged)"
  run $tool sim 900 $PYT tests/test_gpu_sim.py -k "c1_ten or drift_recovery"
done
wide_eval
ffma_chain
cat "$SUM"
