timeout -s KILL 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for r in 1 2; do
bash scripts/ab_libs.sh "" variants/libedbatch_base.so variants/libedbatch_kpsB.so
done
