#!/bin/bash
cd scratch
for mode in 0 1; do
 for st in 2 4 6 8 12; do ./tma_stream $mode $st 32 148; done
 for bk in 64 128; do ./tma_stream $mode 4 $bk 148; ./tma_stream $mode 8 $bk 148; done
 ./tma_stream $mode 4 32 296
 ./tma_stream $mode 8 32 592
done
