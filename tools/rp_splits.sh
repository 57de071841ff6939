# A/B of pass splits with the register-resident 4096-long pass (rpass.cu) against the defaults.
OUT=${OUT:-gpurun_out/rps}
mkdir -p $OUT
RP="FFTC_PASS=rp4096_r16x16x16_c4"
ab() { N=$1; shift; V=""; for s in "$@"; do V="$V s$s:FFTC_PASS_LOGS=$s;$RP"; done; PARITY=${PARITY:-1} timeout 600 python tools/pass_ab.py $N "default:" $V >> $OUT/splits.jsonl 2>> $OUT/err.txt; }
ab $((1<<21)) 12,9
ab $((1<<22)) 12,10 10,12
ab $((1<<23)) 12,11
ab $((1<<24)) 12,12
PARITY=0 ab $((1<<25)) 12,9,4 12,8,5 12,12,1
PARITY=0 ab $((1<<26)) 12,8,6 12,10,4 12,12,2
PARITY=0 ab $((1<<27)) 12,8,7 12,12,3 12,10,5
PARITY=0 ab $((1<<28)) 12,8,8 12,12,4 12,10,6
PARITY=0 ab $((1<<30)) 12,12,6 12,10,8 12,8,10
