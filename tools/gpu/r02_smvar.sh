python tools/dec_instrument.py && (cd paper_2511_14116_b200 && python build.py > /dev/null)
python tools/dec_smvar.py > gpurun_out/smvar_eager.txt 2>&1
DEC_GRAPH=1 python tools/dec_smvar.py > gpurun_out/smvar_graph.txt 2>&1
cat gpurun_out/smvar_eager.txt gpurun_out/smvar_graph.txt
