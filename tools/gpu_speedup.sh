#!/bin/bash
# The paper's speed-up surfaces on one B200 through
# the bench CLI (reference tools/main.cpp run_bench schema): shared vs
# per-system vs cuSPARSE (gtsv/gpsvInterleavedBatch), diffusion (tri) and
# hyperdiffusion (pent, + uniform), Crank-Nicolson steps. -> gpurun_out/speedup/
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/speedup
CLI=paper_1909_04539_b200/bandsolve_b200
N=${SPD_N:-64,128,256,512,1024}
M=${SPD_M:-256,1024,4096,16384,65536}
for mode in exact fast; do
  BANDSOLVE_MODE=$mode timeout 1800 $CLI bench --problem diffusion --variants shared,persystem,cusparse --n $N --m $M \
    --steps ${SPD_STEPS:-200} --out gpurun_out/speedup/diffusion_$mode.csv 2>> gpurun_out/speedup/err.log
  echo "diffusion $mode rc=$?"
  BANDSOLVE_MODE=$mode timeout 1800 $CLI bench --problem hyperdiffusion --variants shared,uniform,persystem,cusparse --n $N --m $M \
    --steps ${SPD_STEPS:-200} --out gpurun_out/speedup/hyperdiffusion_$mode.csv 2>> gpurun_out/speedup/err.log
  echo "hyperdiffusion $mode rc=$?"
done
ls -la gpurun_out/speedup
