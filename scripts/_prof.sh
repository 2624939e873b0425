mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/db.csv; timeout 900 python bench.py --db gpurun_out/db.csv > gpurun_out/bench.json 2> gpurun_out/bench.err
rm -f gpurun_out/r18db.csv; timeout 600 python bench.py --net resnet18 --no-cpu --steps 20 --db gpurun_out/r18db.csv > gpurun_out/r18.json 2> gpurun_out/r18.err
