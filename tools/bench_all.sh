# Every bench line of the round (run on the GPU box from the repo root).
mkdir -p gpurun_out
R=${1:-r2e}
timeout 600 python bench.py > gpurun_out/${R}_c4.json 2> gpurun_out/${R}_c4.err
timeout 600 python bench.py --impl reference > gpurun_out/${R}_c4_ref.json 2>&1
timeout 600 python bench.py --max-trials 1024 > gpurun_out/${R}_c4t1024.json 2> gpurun_out/${R}_c4t1024.err
timeout 600 python bench.py --config 2 > gpurun_out/${R}_c2.json 2> gpurun_out/${R}_c2.err
timeout 600 python bench.py --config 3 > gpurun_out/${R}_c3.json 2> gpurun_out/${R}_c3.err
timeout 600 python bench.py --config 1 > gpurun_out/${R}_c1.json 2> gpurun_out/${R}_c1.err
timeout 600 python bench.py --config 5 > gpurun_out/${R}_c5.json 2> gpurun_out/${R}_c5.err
ls gpurun_out/${R}_*
