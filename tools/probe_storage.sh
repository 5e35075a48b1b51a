#!/usr/bin/env bash
# Storage / GPUDirect Storage probe of a GPU box (development aid, run under gpurun).
O=gpurun_out/probe
mkdir -p $O
{
echo "== nproc / mem"; nproc; free -g
echo "== nvidia-fs"; ls -la /dev/nvidia-fs* 2>&1 | head -3; lsmod 2>/dev/null | grep -i nvidia; cat /proc/driver/nvidia-fs/version 2>&1
echo "== cufile.json"; ls -la /etc/cufile.json /usr/local/cuda/gds 2>&1; grep -v '^\s*//' /etc/cufile.json 2>/dev/null | grep -i "compat\|allow\|posix\|max_direct\|bounce" | head
echo "== mounts"; df -hT . /tmp /root /dev/shm 2>&1; grep -v "cgroup\|proc\|sysfs\|devpts\|mqueue" /proc/mounts | head -30
echo "== block"; lsblk -o NAME,SIZE,TYPE,ROTA,MODEL,MOUNTPOINT 2>&1 | head -20; ls /sys/block 2>&1
echo "== gdscheck"; ls /usr/local/cuda/gds/tools 2>&1; timeout 60 /usr/local/cuda/gds/tools/gdscheck -p 2>&1 | head -60
} > $O/probe.txt 2>&1
for d in "$GRAFT_REPO_ROOT" /tmp /dev/shm; do
  f=$d/_probe_io.bin
  echo "== dd $d" >> $O/probe.txt
  timeout 120 dd if=/dev/zero of=$f bs=16M count=128 oflag=direct 2>&1 | tail -1 >> $O/probe.txt
  timeout 120 dd if=$f of=/dev/null bs=16M iflag=direct 2>&1 | tail -1 >> $O/probe.txt
  timeout 120 dd if=$f of=/dev/null bs=16M 2>&1 | tail -1 >> $O/probe.txt
  rm -f $f
done
timeout 120 python - >> $O/probe.txt 2>&1 <<'EOF'
import ctypes as C
try:
    L = C.CDLL("libcufile.so.0")
except OSError as e:
    L = C.CDLL("/usr/local/cuda/lib64/libcufile.so.0")
class Err(C.Structure):
    _fields_ = [("err", C.c_int), ("cu_err", C.c_int)]
L.cuFileDriverOpen.restype = Err
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
e = L.cuFileDriverOpen()
print("cuFileDriverOpen", e.err, e.cu_err)
v = C.c_int(0)
if hasattr(L, "cuFileGetVersion"):
    print("cuFileGetVersion", L.cuFileGetVersion(C.byref(v)), v.value)
EOF
echo done >> $O/probe.txt
