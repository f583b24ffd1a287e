for i in 1 2; do
for v in default varlib/ocu1.so varlib/ocu4.so; do
if [ $v = default ]; then timeout 300 python tools/c2_probe.py 2>&1 | grep "pk 0" | sed "s#^#$v #"; else FASTPFP_LIB=$v timeout 300 python tools/c2_probe.py 2>&1 | grep "pk 0" | sed "s#^#$v #"; fi
done; done
