# dense kernels with face tiles first (cases that repair edges)
for c in "u16 7 gauss clamp dense 1024" "u16 7 gauss wrap dense 1024" "u8 3 gauss clamp dense 1024" "u8 3 gauss wrap dense 1024" "f32 3 lap wrap auto 1024" "f32 3 lap clamp auto 1024" "f32 3 lap wrap auto 2048"; do
  set -- $c
  timeout 300 python tools/profile_case.py --fmt $1 --k $2 --kernel $3 --mode $4 --path $5 --n $6 --reps 7 2>&1 | tail -1 | sed "s/(all.*//"
done
