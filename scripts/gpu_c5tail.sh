export FHWT_TUNING=1
for i in 1 2; do
python tools/graph_time.py 1 32768 32768 5
python tools/graph_time.py 1 32768 32768 8
FHWT_COOP=0 python tools/graph_time.py 1 32768 32768 8
python tools/graph_time.py 256 2048 2048 5
python tools/graph_time.py 16 8192 8192 5
done
