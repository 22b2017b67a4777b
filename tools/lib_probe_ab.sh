cd /root/repo
for i in 1 2; do
python tools/lib_probe.py tools/var_r01.so paper_1008_1366_b200/libidconv.so
python tools/lib_probe.py paper_1008_1366_b200/libidconv.so --profile
done
