#!/bin/bash
for i in 1 2; do
echo "base: $(timeout 600 python tools/style_batch.py 512x128 4096x128 2>&1 | tail -1)"
echo "lean: $(INET_B200_LEAN=1 timeout 600 python tools/style_batch.py 512x128 4096x128 2>&1 | tail -1)"
done
