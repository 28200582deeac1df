run() { timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 --lora-steps 0 --variant-steps 0 --prof-steps 4 --steps 800 "$@" 2>/dev/null | tail -1; }
for ns in 64 80 96; do
  run --norm-sms $ns --compose-parts fwd
  run --norm-sms $ns --compose-parts bwd
  run --norm-sms $ns --only compose --compose-parts fwd
  run --norm-sms $ns --only compose --compose-parts bwd
done
