cd $GRAFT_REPO_ROOT
for rep in 1 2; do for lib in variants/libaldp_rl.so default; do
if [ "$lib" == "default" ]; then L=""; else L="ALDP_LIB=$lib"; fi
env $L timeout 300 python bench.py --images 4096 --steps 10 --no-cpu > gpurun_out/e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/e.json'));print('$lib', d['e2e']['value'], d['value'])"
done; done
