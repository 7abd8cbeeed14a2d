#!/bin/bash
# Probe the GPU box's storage / host environment (run under gpurun).
set -x
mkdir -p gpurun_out
{
uname -a; nproc; free -g; ulimit -l; cat /proc/cpuinfo | grep "model name" | head -2
lsblk -o NAME,SIZE,TYPE,ROTA,MODEL,MOUNTPOINT,FSTYPE 2>&1
findmnt -D 2>&1 | head -50
df -hT 2>&1
cat /proc/mounts
ls -la /sys/class/nvme/ 2>&1
for d in /sys/class/nvme/nvme*; do echo $d; cat $d/model $d/device/numa_node 2>/dev/null; readlink -f $d/device; done
nvidia-smi; nvidia-smi topo -m
numactl -H 2>&1 || ls /sys/devices/system/node/
python -c "import ctypes; libc=ctypes.CDLL(None,use_errno=True); p=(ctypes.c_char*120)(); r=libc.syscall(425, 8, p); print('io_uring_setup', r, ctypes.get_errno())"
which fio
for dir in /tmp /root /dev/shm /mnt /raid /scratch /data /local $GRAFT_REPO_ROOT; do
  [ -d $dir ] || continue
  echo "=== $dir"; df -hT $dir
  f=$dir/.fp_probe_$$
  timeout 60 dd if=/dev/zero of=$f bs=1M count=2048 oflag=direct conv=fsync 2>&1 | tail -1
  timeout 60 dd if=/dev/zero of=$f bs=1M count=2048 conv=fsync 2>&1 | tail -1
  rm -f $f
done
cat /proc/pressure/io 2>/dev/null
cat /sys/fs/cgroup/io.max 2>/dev/null; cat /sys/fs/cgroup/memory.max 2>/dev/null
} > gpurun_out/probe.txt 2>&1
tail -c 3000 gpurun_out/probe.txt
