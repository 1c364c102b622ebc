for r in 20; do MB_ONLY=store profiles/scripts/microbench/_bin/mb_base $r; profiles/scripts/microbench/_bin/inplace $r; profiles/scripts/microbench/_bin/inplace_tma $r; done
source <(sed -n '/^sample()/,/^}/p' profiles/scripts/microbench/power.sh)
B=profiles/scripts/microbench/_bin; OUT=gpurun_out
sample gen_store env MB_ONLY=store profiles/scripts/microbench/_bin/mb_base 1300
sample gen_inplace profiles/scripts/microbench/_bin/inplace 1300
sample gen_inplace_tma profiles/scripts/microbench/_bin/inplace_tma 1300
