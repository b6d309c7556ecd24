for L in r50.l3.b1.c1 r50.l4.b1.c2; do
python tools/pdl_check.py $L
TP_PDL=0 python tools/pdl_check.py $L
TP_NO_CLUSTER=1 python tools/pdl_check.py $L
done
