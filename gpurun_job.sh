mkdir -p gpurun_out
cp paper_2505_17694_b200/profiles/b200_d128.csv gpurun_out/b200_d128_model.csv
timeout 1200 python -m paper_2505_17694_b200.profile_b200 measure > gpurun_out/profile_measure.log 2>&1; echo "measure exit $?"
cp paper_2505_17694_b200/profiles/b200_d128.csv gpurun_out/b200_d128_measured.csv
tail -3 gpurun_out/profile_measure.log
