TTS=c2 TTS_SOLVERS=cocg timeout 900 python tools/configs_tts.py > gpurun_out/r3j_tts.txt 2>&1
cp profiles/r02_time_to_solution.json gpurun_out/r02_time_to_solution_cocg.json
tail -3 gpurun_out/r3j_tts.txt
