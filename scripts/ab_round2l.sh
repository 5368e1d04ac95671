export PYTHONUNBUFFERED=1
for E in "TVR_PDL=1" "TVR_PDL=0" "TVR_SELL_CTA_TAB=0" "TVR_PDL=0 TVR_SELL_CTA_TAB=0"; do
  echo "== e2e $E"; env $E python scripts/e2e_steps.py 2>&1 | grep -o '"rep[0-9]_[0-9]*": {"evals_per_s": [0-9.]*' 
done
bash scripts/ab_env.sh c3 40 "TVR_PDL=1" "TVR_PDL=0" "TVR_SELL_CTA_TAB=0" "TVR_PDL=0 TVR_SELL_CTA_TAB=0" 2>&1 | awk 'NR%2==0'
