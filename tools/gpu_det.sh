mkdir -p gpurun_out
python tests/scripts/fwd_det.py /tmp/ref.pt
for i in 1 2 3 4 5 6; do
  c=$(( (i % 3) + 1 ))
  SKB_MAX_CTAS=$c python tests/scripts/fwd_det.py /tmp/cap.pt
  python - <<PY
import torch
a=torch.load("/tmp/ref.pt"); b=torch.load("/tmp/cap.pt")
for k in a:
    for nm,x,y in zip(("o","lse","dq","dk","dv"),a[k],b[k]):
        if not torch.equal(x,y): print("DIFF", "$c", k, nm, float((x.double()-y.double()).abs().max()))
print("run $i cap $c done")
PY
done
