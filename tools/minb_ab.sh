#!/bin/bash
for i in 1 2; do
echo "base : $(timeout 600 python tools/style_batch.py 4096x128 2048x128 2>&1 | tail -1)"
echo "minb11: $(INET_B200_MINB=11 timeout 600 python tools/style_batch.py 4096x128 2048x128 2>&1 | tail -1)"
done
