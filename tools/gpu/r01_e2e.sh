OUT=gpurun_out
echo new; python tools/e2e_probe.py 16384 16384 0 0
cp paper_2504_13821_b200/lib/librectri_cu.so /tmp/new.so
cp tools/gpu/old/librectri_cu.so paper_2504_13821_b200/lib/librectri_cu.so
echo old; python tools/e2e_probe.py 16384 16384 0 0
cp /tmp/new.so paper_2504_13821_b200/lib/librectri_cu.so
echo new; python tools/e2e_probe.py 16384 16384 0 0
