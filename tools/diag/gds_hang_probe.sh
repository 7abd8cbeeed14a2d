#!/bin/bash
# Where does cuFileDriverOpen block on the gpurun boxes? Starts the GDS diag
# in the background, waits, dumps every thread's blocked syscall / wchan /
# kernel stack from /proc (no strace/gdb in the image), then kills it.
out=${1:-gpurun_out/gds_probe}
mkdir -p $(dirname $out)
{
  echo "== modules"; lsmod 2>/dev/null | grep -i -E "nvidia|nvme|fs" ; ls -la /dev/nvidia* 2>&1 | head -20
  echo "== /proc/driver/nvidia-fs"; ls /proc/driver/nvidia-fs 2>&1; cat /proc/driver/nvidia-fs/stats 2>&1 | head
  echo "== cufile.json"; grep -n -E "compat|poll|rdma|logging|dir" /etc/cufile.json | head -20
} > $out.env.txt 2>&1
export CUFILE_LOGFILE_PATH=$PWD/$out.cufile.log
export CUFILE_LOGGING_LEVEL=TRACE
export FP_DEBUG_GDS=1 FP_GDS_OPEN_TIMEOUT=60
export CUFILE_SKIP_TOPOLOGY_DETECTION=${CUFILE_SKIP_TOPOLOGY_DETECTION:-true}
[ -n "$PROBE_JSON" ] && export CUFILE_ENV_PATH_JSON=$PWD/$PROBE_JSON
python tools/diag/gds_diag.py c1_tiny ${PROBE_DIR:-/tmp/gds_probe} > $out.diag.log 2>&1 &
pid=$!
sleep 40
{
  echo "== threads of $pid"
  for t in /proc/$pid/task/*; do
    echo "-- $t $(cat $t/comm 2>/dev/null) wchan=$(cat $t/wchan 2>/dev/null)"
    echo "syscall: $(cat $t/syscall 2>/dev/null)"
    cat $t/stack 2>/dev/null | head -12
  done
  echo "== open fds"; ls -la /proc/$pid/fd 2>/dev/null | tail -40
  # the running (spinning) threads: sample their instruction pointers
  gcc -O1 -o /tmp/rip_sample tools/diag/rip_sample.c 2>/dev/null
  for t in /proc/$pid/task/*; do
    if grep -q running $t/syscall 2>/dev/null; then
      echo "== rip samples of ${t##*/}"; /tmp/rip_sample ${t##*/} $pid 12
    fi
  done
} > $out.threads.txt 2>&1
kill -9 $pid 2>/dev/null
wait $pid 2>/dev/null
echo "probe done"
