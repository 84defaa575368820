# Step-time attribution by difference: rerun the bench with one op class skipped
# (TCB_SKIP_OPS, outputs garbage) and print the ms/step saved.
run() {
  TCB_SKIP_OPS="$1" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-max-batch 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1' or 'none', d['ms_per_step'], d.get('clocks'))"
}
run ""
for s in ${SETS:-linear,matmul,matmul_t matmul_pair adam_update_ex,adam_update layer_norm,add_layer_norm \
         layer_norm_dx attention attention_dx colsum embedding,embedding_dx cross_entropy}; do
  run "$s"
done
run ""
