LA_B200_DKDV=pair timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do
echo "fused $(timeout 120 python tools/exp_time.py 2>&1 | tail -1)"
echo "pair  $(LA_B200_DKDV=pair timeout 120 python tools/exp_time.py 2>&1 | tail -1)"
done
