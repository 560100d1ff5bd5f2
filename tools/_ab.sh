# A/B of the library variants in abvar/ against the in-tree build (dev helper)
out=gpurun_out/$1.jsonl; shift
: > $out
python tools/variant_eval.py >> $out
for v in abvar/*.so; do PAGANI_LIB=$v python tools/variant_eval.py >> $out; done
python tools/variant_eval.py >> $out
python tools/variant_table.py $out
