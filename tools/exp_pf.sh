# cross-launch L2 prefetch budget sweep (bench variants, one box)
for mb in 0 8 16 24 32 48; do
  PG_BENCH_PF_MB=$mb timeout 300 python bench.py --steps 640 --warmup 64 --cpu-steps 0 --prefill 0 --decode-batch 0 > gpurun_out/pf_$mb.json 2>gpurun_out/pf_$mb.err || tail -5 gpurun_out/pf_$mb.err
  python -c "import json; d=json.load(open('gpurun_out/pf_$mb.json')); v=d['variants']; print($mb, round(d['value']), round(v['l2_prefetch_next_tok_s']), round(d['e2e']['value']), round(v['l2_prefetch_next_e2e_tok_s']))"
done
